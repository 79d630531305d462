#!/usr/bin/env python
"""Small invocations of the round-2 kernels for compute-sanitizer runs: the fused
covariance / correlation kernel (split-K S = 1, 2, 4 shapes, diagonal and off-diagonal
blocks, ragged edges), the GEMM engine's TMA-store epilogue (gemm with C in, 2mm's lo
output, syrk's off-diagonal tiles), atax's TMEM-x single-pass kernel (threshold lowered so a
small matrix takes it), the chained GEMM launch (PB_CHAIN=1) and the stream-K schedule
(PB_STREAMK=1) — both opt-in, set in the environment before the library loads."""
import os
import sys

os.environ.setdefault("PB_ATAX_ONEPASS_MIN_MB", "0")

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from tests import parity as P  # noqa: E402

torch.cuda.set_device(0)
res = [("cov 132x137", P.check_covariance(132, 137)), ("corr 516x600", P.check_correlation(516, 600)),
       ("cov 1028x1000", P.check_covariance(1028, 1000)),
       ("gemm 300x1028x1200 (TMA epilogue, C in)", P.check_gemm(300, 1028, 1200)),
       ("2mm 300x260x272x292 (TMA epilogue, lo out)", P.check_2mm(300, 260, 272, 292)),
       ("syrk 520x300", P.check_syrk(520, 300)),
       ("atax 300x16388 (TMEM x)", P.check_atax(300, 16388))]
if os.environ.get("PB_CHAIN"):  # (768, 256, 256, 768): both GEMMs on 2-CTA 256 x 256 tiles, no split-K
    res.append(("2mm chain", P.check_2mm(768, 256, 256, 768)))
if os.environ.get("PB_STREAMK"):
    res.append(("gemm streamk", P.check_gemm(300, 1028, 1200)))
for name, r in res:
    print(name, r["ok"], r["err"])
