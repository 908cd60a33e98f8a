TAG=base python tools/sp24_probe2.py > gpurun_out/r2_k5ab.jsonl 2>&1
TAG=mc3 BS_SPLITK_MIN_CHUNKS=3 python tools/sp24_probe2.py >> gpurun_out/r2_k5ab.jsonl 2>&1
TAG=bn256 BS_K5_BN_MAX=256 python tools/sp24_probe2.py >> gpurun_out/r2_k5ab.jsonl 2>&1
TAG=mc3bn256 BS_SPLITK_MIN_CHUNKS=3 BS_K5_BN_MAX=256 python tools/sp24_probe2.py >> gpurun_out/r2_k5ab.jsonl 2>&1
TAG=mc2bn256 BS_SPLITK_MIN_CHUNKS=2 BS_K5_BN_MAX=256 python tools/sp24_probe2.py >> gpurun_out/r2_k5ab.jsonl 2>&1
