"""Tuning aid: per-phase stamps of the fused cov/corr kernel (PB_GRAM_TIMING=1), eager calls."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda", 0)
data = torch.empty(n, n, device=dev)
pbgen.gen_device(data, 5)
out = torch.empty(n, n, device=dev)
ws = pb.workspace("covariance", (n, n), dev)
fl = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for k in ("covariance", "correlation"):
    for it in range(3):
        fl.fill_(1)
        torch.cuda.synchronize()
        print(f"== {k} call {it}", file=sys.stderr, flush=True)
        if k == "covariance":
            pb.pb_covariance(n, n, float(n), data, out, None, ws=ws)
        else:
            pb.pb_correlation(n, n, float(n), 0.1, data, out, None, None, ws=ws)
        torch.cuda.synchronize()
