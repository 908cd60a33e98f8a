# DRAM bytes of the SpMV kernel at the sweep's sparsities (65536^2), against the packed bytes
mkdir -p gpurun_out
for s in 0.5 0.75 0.97; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:spmv_kernel -s 3 -c 1 --csv python tools/ptb_once.py 65536 65536 $s > gpurun_out/r2_sweep_ncu_$s.csv 2>&1; echo "s=$s rc=$?"
done
python - <<'PY' > gpurun_out/r2_sweep_ncu.txt
import sys; sys.path.insert(0, '.')
import paper_1811_00206_b200 as bs, torch
for s in (0.5, 0.75, 0.97):
    k = bs.k_from_sparsity(32, s)
    print(s, k, bs.packed_bytes(65536, 65536, 32, k, torch.float16))
PY
cat gpurun_out/r2_sweep_ncu.txt
