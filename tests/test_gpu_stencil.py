"""GPU parity of the SYCL-Bench stencils (readings R19-R21):
pb_conv2d / pb_conv3d / pb_fdtd_2d through the C ABI against the oracle on pbgen
inputs. conv: componentwise 1e-4 (R8) and border entries untouched bitwise;
fdtd: bitwise equal to the fp32 evaluation of the PolyBench statements and within
1e-4 of max|state| of the fp64 oracle. Sizes span several tiles with ragged tails,
the minimal interiors, and the paper's / bench sizes (sampled rows or planes)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2312_13170_b200 as pb  # noqa: E402
import pbgen  # noqa: E402
from tests import parity as P  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _ok(r):
    assert r["ok"], r


RW9 = list(np.random.default_rng(7).normal(size=9))
RW27 = list(np.random.default_rng(8).normal(size=27))


@pytest.mark.parametrize("ni,nj", [(3, 4), (3, 132), (4, 8), (5, 128), (37, 132), (130, 260), (300, 516), (1030, 1028)])
@pytest.mark.parametrize("w", ["pbgpu", "random"])
def test_conv2d(ni, nj, w):
    _ok(P.check_conv2d(ni, nj, None if w == "pbgpu" else RW9))


@pytest.mark.parametrize("ni,nj,nk", [(3, 3, 4), (3, 4, 132), (5, 9, 12), (12, 17, 132), (33, 11, 260), (70, 20, 128),
                                      (9, 130, 136)])
@pytest.mark.parametrize("w", ["pbgpu", "random"])
def test_conv3d(ni, nj, nk, w):
    _ok(P.check_conv3d(ni, nj, nk, None if w == "pbgpu" else RW27))


@pytest.mark.parametrize("nx,ny,tmax", [(1, 4, 3), (2, 4, 1), (5, 8, 2), (33, 36, 7), (64, 132, 10), (130, 260, 9),
                                        (257, 512, 20)])
def test_fdtd2d(nx, ny, tmax):
    _ok(P.check_fdtd2d(nx, ny, tmax))


def test_fdtd2d_per_step_path():
    """More tiles than SMs: the one-launch-per-step kernel (ping-pong through the workspace)."""
    r = P.check_fdtd2d(2048, 2052, 5)
    _ok(r)
    assert r["bitwise_f32"]


def test_fdtd2d_zero_steps_is_identity():
    ex, ey, hz, f = P.fdtd_inputs(16, 20, 0)
    d = [P.dev(a) for a in (ex, ey, hz)]
    pb.pb_fdtd_2d(0, 16, 20, d[0], d[1], d[2], None)
    for a, b in zip(d, (ex, ey, hz)):
        assert np.array_equal(P.host(a), b)


def test_small_interiors_are_noops():
    A = P.dev(P.H(2, 8, 1))
    B0 = P.H(2, 8, 2)
    dB = P.dev(B0)
    pb.pb_conv2d(2, 8, pbgen.CONV2D_W, A, dB)
    assert np.array_equal(P.host(dB), B0)
    A3 = P.dev(P.H(2 * 5, 8, 1))
    B3 = P.H(2 * 5, 8, 2)
    dB3 = P.dev(B3)
    pb.pb_conv3d(2, 5, 8, pbgen.conv3d_w27(), A3, dB3)
    assert np.array_equal(P.host(dB3), B3)


def test_stencils_deterministic():
    A = P.dev(P.H(64 * 33, 260, 1))
    outs = []
    for _ in range(2):
        B = torch.zeros(64 * 33 * 260, device="cuda")
        pb.pb_conv3d(64, 33, 260, pbgen.conv3d_w27(), A, B)
        outs.append(P.host(B))
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))


def test_stencil_abi_errors():
    A = torch.zeros(16, 16, device="cuda")
    B = torch.zeros(16, 16, device="cuda")
    with pytest.raises(pb.PBError) as e:
        pb.pb_conv2d(16, 16, pbgen.CONV2D_W, A, A)  # output overlaps input
    assert e.value.status == 3
    with pytest.raises(pb.PBError) as e:
        pb.pb_conv2d(16, 15, pbgen.CONV2D_W, A, B)  # nj % 4 != 0
    assert e.value.status == 2
    st = pb.lib().pb_conv2d(16, 16, None, A.data_ptr(), B.data_ptr(), None)  # NULL weights
    assert st == 1
    with pytest.raises(pb.PBError) as e:
        pb.pb_fdtd_2d(3, 16, 16, A, B, A, torch.zeros(3, device="cuda"))  # ex aliases hz
    assert e.value.status == 3
    with pytest.raises(pb.PBError) as e:
        pb.pb_fdtd_2d(-1, 16, 16, A, B, torch.zeros(16, 16, device="cuda"), None)
    assert e.value.status == 1


# ------------------------------------------------------------------ bench / paper sizes
def test_conv2d_paper_size_4096_full():
    _ok(P.check_conv2d(4096, 4096))


def test_conv2d_16384_sampled_rows():
    n = 16384
    A = torch.empty(n, n, device="cuda")
    pbgen.gen_device(A, P.S["A"])
    B = torch.empty(n, n, device="cuda")
    pbgen.gen_device(B, P.S["B"])
    pb.pb_conv2d(n, n, pbgen.CONV2D_W, A, B)
    torch.cuda.synchronize()
    for i in (1, 2, 221, 222, 223, 8191, n - 3, n - 2):  # strip edges included
        Ah = P.host(A[i - 1:i + 2])
        Bin = np.zeros_like(Ah)
        Bin[1] = pbgen.gen_host(1, n, P.S["B"], row0=i)
        r = oracle.conv2d(pbgen.CONV2D_W, Ah, Bin, rows=(1, 2))[0]
        s = oracle.conv2d(pbgen.CONV2D_W, Ah, Bin, rows=(1, 2), absmode=True)[0]
        g = P.host(B[i])
        assert P.cerr(g, r, s) <= P.TOL, i
        assert g[0] == Bin[1][0] and g[-1] == Bin[1][-1]
    for i in (0, n - 1):  # border rows untouched
        assert np.array_equal(P.host(B[i]), pbgen.gen_host(1, n, P.S["B"], row0=i)[0])


def test_conv3d_bench_size_1024_sampled_planes():
    n = 1024
    A = torch.empty(n * n, n, device="cuda")
    pbgen.gen_device(A, P.S["A"])
    B = torch.empty(n * n, n, device="cuda")
    pbgen.gen_device(B, P.S["B"])
    w = pbgen.conv3d_w27()
    pb.pb_conv3d(n, n, n, w, A, B)
    torch.cuda.synchronize()
    for p0 in (1, 500, n - 2):
        Ah = P.host(A[(p0 - 1) * n:(p0 + 2) * n]).reshape(3, n, n)
        Bin = np.zeros_like(Ah)
        Bin[1] = pbgen.gen_host(n, n, P.S["B"], row0=p0 * n)
        r = oracle.conv3d(w, Ah, Bin, planes=(1, 2))[0]
        s = oracle.conv3d(w, Ah, Bin, planes=(1, 2), absmode=True)[0]
        g = P.host(B[p0 * n:(p0 + 1) * n])
        assert P.cerr(g, r, s) <= P.TOL
        m = P._border_mask((n, n))
        assert np.array_equal(g[m], Bin[1][m])
    # border planes untouched
    g0 = P.host(B[0:n])
    assert np.array_equal(g0, pbgen.gen_host(n, n, P.S["B"], row0=0))


def test_fdtd2d_paper_size_1024_500_steps():
    r = P.check_fdtd2d(1024, 1024, 500)
    _ok(r)
    assert r["bitwise_f32"]


# ------------------------------------------------------------------ gramschmidt (R22)
@pytest.mark.parametrize("m,n", [(1, 1), (5, 1), (4, 4), (37, 20), (132, 132), (300, 149), (149, 148), (517, 300),
                                 (1024, 1024)])
def test_gramschmidt(m, n):
    """m >= n: with n > m the columns k >= m are linearly dependent, R[k][k] is
    rounding noise and Q[:, k] = noise / noise (Inf/NaN or arbitrary), on both sides."""
    _ok(P.check_gramschmidt(m, n))


def test_gramschmidt_global_column_path():
    """m * ceil(n / SMs) * 8 B > 200 KiB: the owned columns stay in the workspace (L2)."""
    _ok(P.check_gramschmidt(8192, 600))


def test_gramschmidt_deterministic():
    m, n = 256, 200
    A = P.H(m, n, 1)
    outs = []
    for _ in range(2):
        dA, dR, dQ = P.dev(A), torch.zeros(n, n, device="cuda"), torch.zeros(m, n, device="cuda")
        pb.pb_gramschmidt(m, n, dA, dR, dQ)
        outs.append([P.host(t).view(np.uint32) for t in (dA, dR, dQ)])
    assert all(np.array_equal(a, b) for a, b in zip(*outs))


def test_next_rows_on_a_side_stream():
    """Every NEXT-3 entry point enqueues on the caller's stream (not the default one)."""
    st = torch.cuda.Stream()
    A = P.dev(P.H(260, 516, 1))
    B = torch.zeros(260, 516, device="cuda")
    ex, ey, hz, f = P.fdtd_inputs(130, 132, 9)
    d = [P.dev(a) for a in (ex, ey, hz)]
    G = P.dev(P.H(200, 132, 1))
    R, Q = torch.zeros(132, 132, device="cuda"), torch.zeros(200, 132, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        pb.pb_conv2d(260, 516, pbgen.CONV2D_W, A, B)
        pb.pb_fdtd_2d(9, 130, 132, d[0], d[1], d[2], P.dev(f))
        pb.pb_gramschmidt(200, 132, G, R, Q)
    st.synchronize()
    r = oracle.conv2d(pbgen.CONV2D_W, P.H(260, 516, 1), np.zeros((260, 516), np.float32))
    s = oracle.conv2d(pbgen.CONV2D_W, P.H(260, 516, 1), np.zeros((260, 516), np.float32), absmode=True)
    assert P.cerr(P.host(B), r, s) <= P.TOL
    r32 = oracle.fdtd2d(9, ex, ey, hz, f, f32=True)
    assert all(np.array_equal(P.host(a).view(np.uint32), b.view(np.uint32)) for a, b in zip(d, r32))
    rA, rR, rQ = oracle.gramschmidt(P.H(200, 132, 1))
    assert (np.abs(P.host(Q) - rQ) / np.abs(rQ).max(0)).max() <= P.TOL


def test_conv_zero_weights():
    A = P.dev(P.H(37 * 9, 132, 1))
    B = P.dev(P.H(37 * 9, 132, 2))
    pb.pb_conv3d(37, 9, 132, [0.0] * 27, A, B)
    g = P.host(B).reshape(37, 9, 132)
    assert np.all(g[1:-1, 1:-1, 1:-1] == 0)


@pytest.mark.parametrize("G", [2, 3, 8])
def test_conv_row_blocks_equal_whole(G):
    """Row-block sharding of the convolutions needs no new entry point and no data-path
    exchange: rank g calls pb_conv2d / pb_conv3d on its rows (planes) plus one halo row
    (plane) on each side; the local call leaves its first and last rows unwritten, which
    are exactly the halo. The union equals the single call bitwise (per-point FMA order
    is independent of the decomposition)."""
    ni, nj = 1000, 1028
    A = P.dev(P.H(ni, nj, 1))
    whole = P.dev(P.H(ni, nj, 2))
    pb.pb_conv2d(ni, nj, pbgen.CONV2D_W, A, whole)
    sharded = P.dev(P.H(ni, nj, 2))
    for g in range(G):
        r0, r1 = pb.pb_row_partition(ni, G, g)
        lo, hi = max(r0 - 1, 0), min(r1 + 1, ni)
        pb.pb_conv2d(hi - lo, nj, pbgen.CONV2D_W, A[lo:hi], sharded[lo:hi])
    assert np.array_equal(P.host(whole).view(np.uint32), P.host(sharded).view(np.uint32))
    n3, nj3, nk3 = 67, 33, 260
    A3 = P.dev(P.H(n3 * nj3, nk3, 1)).view(n3, nj3, nk3)
    w3 = torch.zeros(n3, nj3, nk3, device="cuda")
    s3 = torch.zeros(n3, nj3, nk3, device="cuda")
    pb.pb_conv3d(n3, nj3, nk3, pbgen.conv3d_w27(), A3, w3)
    for g in range(G):
        p0, p1 = pb.pb_row_partition(n3, G, g)
        lo, hi = max(p0 - 1, 0), min(p1 + 1, n3)
        pb.pb_conv3d(hi - lo, nj3, nk3, pbgen.conv3d_w27(), A3[lo:hi], s3[lo:hi])
    assert np.array_equal(P.host(w3).view(np.uint32), P.host(s3).view(np.uint32))


@pytest.mark.parametrize("variant", [0, 1])
def test_conv_variants(variant):
    """pb_conv2d_variant / pb_conv3d_variant (0: one thread per point, global loads; 1:
    production) against the oracle, borders untouched."""
    ni, nj = 67, 132
    A, B0 = P.H(ni, nj, 1), P.H(ni, nj, 2)
    dB = P.dev(B0)
    pb.pb_conv2d_variant(variant, ni, nj, pbgen.CONV2D_W, P.dev(A), dB)
    r, s = oracle.conv2d(pbgen.CONV2D_W, A, B0), oracle.conv2d(pbgen.CONV2D_W, A, B0, absmode=True)
    g = P.host(dB)
    assert P.cerr(g, r, s) <= P.TOL
    n3 = (13, 11, 132)
    A3 = P.H(n3[0] * n3[1], n3[2], 1).reshape(n3)
    B3 = P.H(n3[0] * n3[1], n3[2], 2).reshape(n3)
    dB3 = P.dev(B3)
    pb.pb_conv3d_variant(variant, *n3, pbgen.conv3d_w27(), P.dev(A3), dB3)
    r, s = oracle.conv3d(pbgen.conv3d_w27(), A3, B3), oracle.conv3d(pbgen.conv3d_w27(), A3, B3, absmode=True)
    assert P.cerr(P.host(dB3), r, s) <= P.TOL


@pytest.mark.parametrize("variant", [0, 1])
def test_gramschmidt_variants(variant):
    """pb_gramschmidt_variant (0: PolyBench-GPU three-launches-per-column shape; 1:
    production) against the oracle (reading R22)."""
    m, n = 300, 149
    A = P.H(m, n, 1)
    dA, dR, dQ = P.dev(A), torch.zeros(n, n, device="cuda"), torch.zeros(m, n, device="cuda")
    pb.pb_gramschmidt_variant(variant, m, n, dA, dR, dQ)
    rA, rR, rQ = oracle.gramschmidt(A)
    gA, gR, gQ = P.host(dA), P.host(dR), P.host(dQ)
    cn = np.sqrt((A.astype(np.float64) ** 2).sum(0))
    up = np.triu(np.ones((n, n), bool))
    assert (np.abs(gQ - rQ) / np.abs(rQ).max(0)).max() <= P.TOL
    assert (np.abs(gA - rA) / np.abs(rA).max(0)).max() <= P.TOL
    assert (np.abs(gR - rR) / cn[None, :])[up].max() <= P.TOL


def test_new_entry_points_reject_bad_arguments():
    """Validation before any enqueue (include/pb.h conventions) for the entry points added
    this round: aliasing, row-range rules, unknown variants."""
    A = torch.zeros(256, 256, device="cuda")
    R = torch.zeros(256, 256, device="cuda")
    with pytest.raises(pb.PBError) as e:
        pb.pb_gramschmidt(256, 256, A, R, A)  # Q aliases A
    assert e.value.status == 3
    with pytest.raises(pb.PBError) as e:
        pb.pb_covariance_rows(256, 256, 256.0, 64, 256, A, R[:192])  # r0 not a multiple of 128
    assert e.value.status == 1
    with pytest.raises(pb.PBError) as e:
        pb.pb_correlation_rows(256, 256, 256.0, 0.1, 128, 300, A, R)  # r1 > m
    assert e.value.status == 1
    with pytest.raises(pb.PBError) as e:
        pb.pb_conv2d_variant(7, 256, 256, pbgen.CONV2D_W, A, R)
    assert e.value.status == 1
    with pytest.raises(pb.PBError) as e:
        pb.pb_gramschmidt_variant(5, 256, 256, A, R, torch.zeros(256, 256, device="cuda"))
    assert e.value.status == 1


def test_conv3d_large_grid_tile_paths_ragged():
    """The 16-row conv3d tiles (16 x 256 when rows have >= 256 columns, else 16 x 128) are
    taken for grids of >= 2^28 points; PB_C3_RPW=2 forces them on small ragged grids (rows
    and columns not multiples of the tile, both weight masks) in a subprocess, since the
    library reads the variable once per process."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r); from tests import parity as P; import pbgen;"
            "rw = [((k * 7) %% 11 - 5) / 8.0 for k in range(27)];"
            "res = [P.check_conv3d(20, 37, 260), P.check_conv3d(18, 35, 132), P.check_conv3d(19, 33, 300, rw),"
            "       P.check_conv3d(17, 40, 140, rw)];"
            "bad = [r for r in res if not r['ok']]; print('bad', bad); sys.exit(1 if bad else 0)" % root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, PB_C3_RPW="2"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
