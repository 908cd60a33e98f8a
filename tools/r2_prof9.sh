python -m pytest tests -m gpu -q > gpurun_out/r2_gpu9.log 2>&1
python tools/direct_probe.py > gpurun_out/r2_direct4.jsonl 2>&1
python bench.py > gpurun_out/r2_bench9.json 2> gpurun_out/r2_bench9.err
