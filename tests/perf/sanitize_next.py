#!/usr/bin/env python
"""Small invocations of the NEXT-3 kernels for compute-sanitizer runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from tests import parity as P  # noqa: E402

torch.cuda.set_device(0)
for name, r in (("conv2d", P.check_conv2d(37, 1032)), ("conv3d", P.check_conv3d(12, 17, 260)),
                ("fdtd_2d", P.check_fdtd2d(130, 260, 9)), ("gramschmidt", P.check_gramschmidt(132, 100))):
    print(name, r["ok"], r["err"])
