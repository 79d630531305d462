#!/usr/bin/env python
"""One call of a stencil at its bench size (for ncu captures): conv2d 16384^2,
conv3d 1024^3, fdtd_2d 1024^2 (tmax steps), gramschmidt 1024^2.
usage: python scripts/stencil_one.py conv2d|conv3d|fdtd_2d|gramschmidt [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402

S = pbgen.STREAM
k = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)


def gen(shape, stream):
    t = torch.empty(*shape, device=dev)
    pbgen.gen_device(t.view(-1, shape[-1]), stream)
    return t


if k == "conv2d":
    n = 16384
    A, B = gen((n, n), S["A"]), gen((n, n), S["B"])
    fn = lambda: pb.pb_conv2d(n, n, pbgen.CONV2D_W, A, B)  # noqa: E731
elif k == "conv3d":
    n = 1024
    A, B = gen((n, n, n), S["A"]), gen((n, n, n), S["B"])
    fn = lambda: pb.pb_conv3d(n, n, n, pbgen.conv3d_w27(), A, B)  # noqa: E731
elif k == "fdtd_2d":
    n, T = 1024, 20
    ex, ey, hz = gen((n, n), S["ex"]), gen((n, n), S["ey"]), gen((n, n), S["hz"])
    f = gen((1, T), S["fict"]).view(-1)
    ws = pb.workspace("fdtd_2d", (n, n), dev)
    fn = lambda: pb.pb_fdtd_2d(T, n, n, ex, ey, hz, f, ws)  # noqa: E731
elif k == "gramschmidt":
    n = 1024
    A = gen((n, n), S["A"])
    R = torch.zeros(n, n, device=dev)
    Q = torch.zeros(n, n, device=dev)
    A0 = A.clone()
    ws = pb.workspace("gramschmidt", (n, n), dev)

    def fn():
        A.copy_(A0)
        pb.pb_gramschmidt(n, n, A, R, Q, ws)
for _ in range(reps):
    fn()
torch.cuda.synchronize()
print("ok", k)
