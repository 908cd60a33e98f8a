# Round-2 final evidence pass: full bench line, launch list of the bench command, one ncu --set full of the SpMV
mkdir -p gpurun_out
bash tools/gpu_profile.sh r2s4
python tools/ncu_summary.py gpurun_out/prof_spmv_r2s4.ncu-rep "SpMV 65536^2 s=0.9 (bench launch), round 2 final" > gpurun_out/r2s4_spmv_ncu.md 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_r2s4.json 2> gpurun_out/bench_reference_r2s4.err; echo "ref rc=$?"
