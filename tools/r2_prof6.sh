python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu6.log 2>&1
python tools/direct_probe.py > gpurun_out/r2_direct.jsonl 2>&1
BS_DIRECT_ROW_BYTES=8192 python tools/direct_probe.py > gpurun_out/r2_direct_8k.jsonl 2>&1
