"""Per-rank GEMM shape at G = 4 / 8 (rows = 1024 / 512 of 4096 x 4096 x 4096) under the
current plan or a forced split-K (PB_UMMA_KSPLIT, read once per process)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_13170_b200 as pb
import pbgen
dev = torch.device("cuda", 0)
def g(r, c, s):
    t = torch.empty(r, c, device=dev); pbgen.gen_device(t, s); return t
def timed(fn, reps=10):
    fn(); torch.cuda.synchronize()
    st = torch.cuda.Stream(); gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st): fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
N = 4096
A, B = g(N, N, 1), g(N, N, 2)
for rows in (512, 1024):
    C = torch.empty(rows, N, device=dev)
    ws = pb.workspace("gemm", (rows, N, N), dev)
    t = timed(lambda: pb.pb_gemm(rows, N, N, 1.0, 0.0, C, A[:rows], B, ws=ws))
    print("KS", os.environ.get("PB_UMMA_KSPLIT", "plan"), os.environ.get("PB_UMMA_TILE", "-"), rows, round(t * 1e3, 1), "us",
          round(2 * rows * N * N / t / 1e9, 1), "TF/s")
