"""BASELINE configs[2] on its own: bench.c3_targets (sigma sweep at N=2^22,
Metropolis bias vs B, rejection acceptance) -> profiles/<tag>_c3_sweep.json."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1301_4019_b200 as pf  # noqa: E402

pf.config.check = False
t0 = time.time()
res = bench.c3_targets(pf, torch, torch.device("cuda"), torch.cuda.current_stream())
res["wall_s"] = time.time() - t0
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = os.path.join(ROOT, "gpurun_out", f"{tag}_c3_sweep.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
with open(out, "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps(res)[:3000])
