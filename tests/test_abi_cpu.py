"""CPU-side checks of the boundary (no GPU needed): libpb loads, exports every
function include/pb.h declares, the binding declares the same set, the
host-only entry points behave, and the product path never touches oracle/."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2312_13170_b200 as pb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "pb.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", txt))


def test_header_symbols_exported_and_bound():
    names = header_functions()
    assert len(names) >= 20
    L = ctypes.CDLL(pb.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n
    assert names == set(pb.ABI_FUNCTIONS), names ^ set(pb.ABI_FUNCTIONS)
    out = subprocess.check_output(["nm", "-D", "--defined-only", pb.LIB_PATH]).decode()
    exported = set(re.findall(r" T (pb_[a-z0-9_]+)", out))
    assert names <= exported


def test_libpb_is_sm100a_and_has_tcgen05():
    out = subprocess.check_output(["cuobjdump", "--list-elf", pb.LIB_PATH]).decode()
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", pb.LIB_PATH]).decode()
    assert "UTCHMMA" in sass or "UTCMMA" in sass or re.search(r"UTC\w*MMA", sass)
    assert "UTMALDG" in sass  # TMA tile loads
    assert "LDTM" in sass     # tcgen05.ld


def test_status_and_version():
    assert pb.lib().pb_status_str(0) == b"PB_OK"
    assert pb.lib().pb_status_str(3) == b"PB_ERR_ALIAS"
    assert "sm_100a" in pb.pb_version()


def test_workspace_sizes():
    # raw-hi split: one lo array per operand (A, and B as stored)
    assert pb.workspace_size("gemm", (128, 128, 128)) == 2 * 128 * 128 * 4
    assert pb.workspace_size("gemm", (7, 4, 5)) >= 4 * (7 * 8 + 5 * 4)
    assert pb.workspace_size("syr2k", (8192, 8192)) >= 2 * 8192 * 8192 * 4  # + split-K partials
    for k, d in [("2mm", (4, 4, 4, 4)), ("3mm", (4, 4, 4, 4, 4)), ("covariance", (8, 9)),
                 ("correlation", (8, 9)), ("atax", (5, 8)), ("bicg", (8, 5)), ("mvt", (8,)),
                 ("gesummv", (8,)), ("syrk_rows", (256, 8, 128, 256)), ("matvec_partial", (3, 8))]:
        assert pb.workspace_size(k, d) % 256 == 0
    with pytest.raises(pb.PBError):
        pb.workspace_size("nope", (1,))
    with pytest.raises(pb.PBError):
        pb.workspace_size("gemm", (1, 2))


@pytest.mark.parametrize("rows,G,tri,align", [(4096, 8, False, 128), (8192, 8, True, 128),
                                               (1000, 3, False, 1), (520, 3, True, 128), (32768, 7, False, 4)])
def test_row_partition(rows, G, tri, align):
    bounds = [pb.pb_row_partition(rows, G, g, tri, align) for g in range(G)]
    assert bounds[0][0] == 0 and bounds[-1][1] == rows
    for (b0, e0), (b1, e1) in zip(bounds, bounds[1:]):
        assert e0 == b1 and b0 <= e0
    for b, e in bounds:
        assert b % align == 0
    if tri:  # areas of the lower-triangle bands are balanced to within one align band
        areas = [(e * (e + 1) - b * (b + 1)) / 2 for b, e in bounds]
        assert max(areas) - min(areas) <= 2 * align * rows


def test_abi_rejects_without_gpu_or_bad_args():
    # invalid dims are rejected before any CUDA call
    st = pb.lib().pb_gemm(0, 4, 4, 1.0, 1.0, None, None, None, None, 0, None)
    assert st == 1
    st = pb.lib().pb_row_partition(10, 0, 0, 0, 1, ctypes.byref(ctypes.c_int()), ctypes.byref(ctypes.c_int()))
    assert st == 1
    assert pb.lib().pb_last_error()


def test_product_path_never_uses_oracle():
    pkg = os.path.join(ROOT, "paper_2312_13170_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), f
                assert "pb_oracle" not in src and "libpb_oracle" not in src, f
    out = subprocess.check_output(["nm", "-D", pb.LIB_PATH]).decode()
    assert "pbo_" not in out
    ldd = subprocess.check_output(["ldd", pb.LIB_PATH]).decode()
    assert "oracle" not in ldd and "pbgen" not in ldd


def test_dist_workspace_sizes_cpu():
    """pb_workspace_size for the multi-GPU entry points ("<k>_dist": dims + {nranks, rank}):
    host-only, so it runs without a GPU or NCCL."""
    import paper_2312_13170_b200 as pb
    n = 32768
    # atax: partial vector (n floats, 256-B aligned) + the local single-pass workspace
    for G in (1, 2, 8):
        for g in range(G):
            r0, r1 = pb.pb_row_partition(n, G, g, False, 4)
            need = pb.workspace_size("atax_dist", (n, n, G, g))
            assert need >= n * 4 + pb.workspace_size("atax", (r1 - r0, n))
            assert pb.workspace_size("gesummv_dist", (n, G, g)) == pb.workspace_size("gesummv_rows", (r1 - r0, n))
            assert pb.workspace_size("mvt_dist", (n, G, g)) >= 2 * n * 4
    # the GEMM family needs at least its local shard's workspace
    assert pb.workspace_size("gemm_dist", (4096, 4096, 4096, 2, 1)) >= pb.workspace_size("gemm", (2048, 4096, 4096))
    assert pb.workspace_size("3mm_dist", (4096,) * 5 + (4, 3)) >= pb.workspace_size("gemm", (1024, 4096, 4096))
    r0, r1 = pb.pb_row_partition(8192, 4, 3, 2, 256)
    assert pb.workspace_size("syr2k_dist", (8192, 8192, 4, 3)) == pb.workspace_size("syr2k_rows", (8192, 8192, r0, r1))
    # covariance / correlation, observations split: the rank's sums gather buffer [G][2][m]
    # doubles + its centred transpose (m x ceil4(obs)) + the m x m partial Gram + pb_syrk_full's
    m, nobs = 2048, 2048
    for G in (1, 2, 8):
        for g in range(G):
            o0, o1 = pb.pb_row_partition(nobs, G, g, False, 32)
            nl = (o1 - o0 + 3) // 4 * 4
            need = pb.workspace_size("covariance_dist", (m, nobs, G, g))
            assert need == pb.workspace_size("correlation_dist", (m, nobs, G, g))
            assert need >= G * 2 * m * 8 + m * nl * 4 + m * m * 4 + pb.workspace_size("syrk_full", (m, nl))
    for bad in [("covariance_dist", (m, nobs, 2, 2)), ("covariance_dist", (m, nobs)), ("correlation_dist", (0, 4, 1, 0))]:
        with pytest.raises(pb.PBError):
            pb.workspace_size(*bad)
    for bad in [("atax_dist", (n, n, 2, 2)), ("atax_dist", (n, n, 0, 0)), ("atax_dist", (n, n)),
                ("nope_dist", (1, 1, 1)), ("gemm_dist", (0, 4, 4, 1, 0))]:
        with pytest.raises(pb.PBError):
            pb.workspace_size(*bad)


def test_row_partition_syrk_cost_balance():
    """triangular = 2 (syrk/syr2k): blocks tile [0, n) in order, aligned, and the
    max per-rank cost (triangle area + 210 * end, the split of A[0:end]) is lower
    than with the pure area balance (triangular = 1)."""
    import paper_2312_13170_b200 as pb

    def cost(b, e):
        return (e * e - b * b) / 2 + 210.0 * e
    for n in (8192, 4096):
        for G in (2, 4, 8):
            worst = {}
            for mode in (1, 2):
                bounds = [pb.pb_row_partition(n, G, g, mode, 256) for g in range(G)]
                assert bounds[0][0] == 0 and bounds[-1][1] == n
                assert all(bounds[g][1] == bounds[g + 1][0] for g in range(G - 1))
                assert all(b % 256 == 0 for b, _ in bounds)
                worst[mode] = max(cost(b, e) for b, e in bounds)
            assert worst[2] <= 1.02 * worst[1]  # block snapping to 256 rows limits small G
    b = [pb.pb_row_partition(8192, 8, g, 2, 256) for g in range(8)]
    assert max(cost(*x) for x in b) < 0.93 * max(cost(*pb.pb_row_partition(8192, 8, g, 1, 256)) for g in range(8))
