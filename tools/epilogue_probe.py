"""Time the fused layer epilogue legs (bench.py epilogue_rows) alone: python tools/epilogue_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1811_00206_b200 as bs  # noqa: E402

sys.argv = sys.argv[:1]
a = bench.parse()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
for r in bench.epilogue_rows(a, bs, l2)["epilogue"]:
    print(json.dumps(r))
