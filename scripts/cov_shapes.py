"""PB_TIMELINE helper: eager covariance calls at (m, n) shapes given on the command line."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402

dev = torch.device("cuda", 0)
for arg in sys.argv[1:]:
    m, n = map(int, arg.split("x"))
    data = torch.empty(n, m, device=dev)
    pbgen.gen_device(data, 5)
    cov = torch.empty(m, m, device=dev)
    ws = pb.workspace("covariance", (m, n), dev)
    for _ in range(3):
        print(f"m={m} n={n}", file=sys.stderr, flush=True)
        pb.pb_covariance(m, n, float(n), data, cov, None, ws=ws)
    torch.cuda.synchronize()
