import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_13170_b200 as pb
import pbgen
dev = torch.device("cuda", 0)
def g(r, c, s):
    t = torch.empty(r, c, device=dev); pbgen.gen_device(t, s); return t
for (M, N, K) in ((512, 4096, 4096), (1024, 1024, 1024), (4096, 4096, 4096)):
    A, B, C = g(M, K, 1), g(K, N, 2), g(M, N, 3)
    ws = pb.workspace("gemm", (M, N, K), dev)
    for _ in range(3):
        pb.pb_gemm(M, N, K, 1.5, 1.2, C, A, B, ws=ws)
        torch.cuda.synchronize()
    print("shape", M, N, K, flush=True)
