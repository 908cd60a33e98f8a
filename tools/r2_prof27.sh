mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench27.json 2> gpurun_out/r2_bench27.err; echo "bench rc=$?"
tail -2 gpurun_out/r2_bench27.err
