# ncu of K5 at 16384^2 N = 1024, RT = 2 and RT = 1
mkdir -p gpurun_out
for rt in 2 1; do
BS_K5_RT=$rt timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm24_kernel -s 2 -c 1 -o gpurun_out/r2_k5_n1024_rt$rt python tools/k5_once.py 16384 16384 1024 > gpurun_out/r2_k5_ncu_rt$rt.log 2>&1; echo "ncu rt=$rt rc=$?"
done
