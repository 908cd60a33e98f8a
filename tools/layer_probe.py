"""Time the paper's latency-regime layers (bench.py layer_rows) without the rest of the bench:
python tools/layer_probe.py [f16|bf16]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1811_00206_b200 as bs  # noqa: E402

sys.argv = [sys.argv[0]] + (["--dtype", sys.argv[1]] if len(sys.argv) > 1 else [])
a = bench.parse()
hbm = bench.peaks()[0]
l2 = torch.cuda.get_device_properties(0).L2_cache_size
for r in bench.layer_rows(a, bs, hbm, l2)["layers"]:
    print(json.dumps(r))
