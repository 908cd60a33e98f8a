mkdir -p gpurun_out
for n in 1024 128; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm24_pair -s 2 -c 1 -o gpurun_out/r2_k5_pair2_n$n python tools/k5_once.py 16384 16384 $n > gpurun_out/r2_k5_pair2_ncu_$n.log 2>&1; echo "ncu rc=$?"
done
