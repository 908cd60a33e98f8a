# Session-3 baseline: full GPU suite + bench line + direct-kernel A/B on HEAD.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu16.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2_gpu16.log
timeout 600 python bench.py > gpurun_out/r2_bench16.json 2> gpurun_out/r2_bench16.err; echo "bench rc=$?"
timeout 300 python tools/direct_probe.py > gpurun_out/r2_direct16.jsonl 2>&1
