# Round-2 final pass on HEAD: full GPU suite, smoke, bench line, launch list, ncu of the SpMV, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu65.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_gpu65.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke65.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke65.log
bash tools/gpu_profile.sh r2s7
python tools/ncu_summary.py gpurun_out/prof_spmv_r2s7.ncu-rep "SpMV 65536^2 s=0.9 (bench launch), round 2 final" > gpurun_out/r2s7_spmv_ncu.md 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_r2s7.json 2> gpurun_out/bench_reference_r2s7.err; echo "ref rc=$?"
