"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same pbgen inputs. Sizes span several 128x128 tiles with ragged tails; the
exactness, determinism and precision-discriminator pins (P1, P32, P34 of
SURVEY.md §8(c)) and the ABI's error behaviour are checked here too.
Full BASELINE.json-size checks live in test_gpu_fullsize.py.
"""
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
    assert r["ok"], {k: v for k, v in r.items() if k not in ("g", "r")}


# ------------------------------------------------------------------ generator
def test_pbgen_device_matches_host_bitwise():
    for mode in (pbgen.U01, pbgen.INT8, pbgen.U01 | pbgen.SYM):
        t = torch.empty(77, 132, device="cuda")
        pbgen.gen_device(t, 3, mode=mode, scale=0.5, offset=-0.25, row0=5, ld=132)
        h = pbgen.gen_host(77, 132, 3, mode=mode, scale=0.5, offset=-0.25, row0=5, ld=132)
        assert np.array_equal(P.host(t).view(np.uint32), h.view(np.uint32))


# ------------------------------------------------------------------ gemm family
@pytest.mark.parametrize("ni,nj,nk", [(128, 128, 32), (128, 128, 128), (7, 4, 4), (129, 132, 260), (130, 132, 128),
                                      (300, 516, 388), (1000, 1024, 1000), (640, 384, 2052)])
def test_gemm(ni, nj, nk):
    _ok(P.check_gemm(ni, nj, nk))


@pytest.mark.parametrize("alpha,beta", [(1.5, 0.0), (0.0, 1.2), (-2.0, 0.5), (1.0, 1.0)])
def test_gemm_alpha_beta(alpha, beta):
    _ok(P.check_gemm(257, 260, 300, alpha, beta))


# small-problem path (ni*nj*nk <= 2^21: one SIMT launch): ragged tiles, several K strips + tail
@pytest.mark.parametrize("ni,nj,nk,alpha,beta", [(100, 36, 260, 1.5, 1.2), (33, 20, 12, 1.5, 1.2), (1, 4, 4, 2.0, 0.5),
                                                 (17, 128, 516, -1.0, 0.0), (128, 128, 128, 0.0, 1.2)])
def test_gemm_small_path(ni, nj, nk, alpha, beta):
    _ok(P.check_gemm(ni, nj, nk, alpha, beta))


def test_gemm_small_path_beta0_ignores_C():
    """beta == 0: C is write-only (include/pb.h), so NaN in C must not propagate."""
    import paper_2312_13170_b200 as pb
    A, B = pbgen.gen_host(64, 96, 1), pbgen.gen_host(96, 32, 2)
    C = P.dev(np.full((64, 32), np.nan, dtype=np.float32))
    pb.pb_gemm(64, 32, 96, 1.5, 0.0, C, P.dev(A), P.dev(B))
    r = oracle.gemm(1.5, 0.0, np.zeros((64, 32), np.float32), A, B)
    g = P.host(C)
    assert np.isfinite(g).all() and np.max(np.abs(g - r) / np.abs(r)) <= P.TOL


def test_gemm_integer_inputs_bitwise_P1():
    """values in {0..7}: hi = x, lo = 0, every product and partial sum exact
    in fp32 -> the tensor-core path equals the oracle bit for bit."""
    r = P.check_gemm(384, 260, 1024, alpha=1.5, beta=0.5, mode=pbgen.INT8)
    assert np.array_equal(r["g"].astype(np.float64), r["r"])


def test_gemm_run_to_run_deterministic_P32():
    A = torch.from_numpy(P.H(512, 516, 1)).cuda()
    B = torch.from_numpy(P.H(516, 384, 2)).cuda()
    C0 = torch.from_numpy(P.H(512, 384, 3)).cuda()
    outs = []
    for _ in range(3):
        C = C0.clone()
        pb.pb_gemm(512, 384, 516, 1.5, 1.2, C, A, B)
        outs.append(P.host(C))
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_gemm_mixed_whole_and_split_tiles_deterministic():
    """A plan with whole tiles AND split-K units (2560 x 2048: 80 tiles of 256 x 256 for 74 SM
    pairs -> 74 whole tiles first, then the 6 remainder tiles split along K, summed by the
    last arriver in split order): parity with the oracle and bitwise run-to-run equality."""
    M, N, K = 2560, 2048, 512
    A, B, C0 = P.H(M, K, 1), P.H(K, N, 2), P.H(M, N, 3)
    dA, dB = P.dev(A), P.dev(B)
    outs = []
    for _ in range(3):
        C = P.dev(C0)
        pb.pb_gemm(M, N, K, 1.5, 1.2, C, dA, dB)
        outs.append(P.host(C))
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    r = oracle.gemm(1.5, 1.2, C0, A, B)
    assert P.cerr(outs[0], r, np.abs(r)) <= P.TOL  # non-negative inputs: the scale is |r| (R8)


def test_gemm_precision_discriminator_P34():
    """centred inputs U[-1/2,1/2): 3xTF32 must stay at fp32-level error
    (<= 2e-6 of |A||B|), which a silent 1xTF32 path (~1e-5) would fail."""
    for nk in (2048, 4096):
        A = P.H(256, nk, 1, offset=-0.5)
        B = P.H(nk, 256, 2, offset=-0.5)
        C = np.zeros((256, 256), np.float32)
        dC = P.dev(C)
        pb.pb_gemm(256, 256, nk, 1.0, 0.0, dC, P.dev(A), P.dev(B))
        g = P.host(dC)
        r = oracle.gemm(1.0, 0.0, C, A, B)
        scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
        assert np.max(np.abs(g - r) / scale) <= 2e-6


@pytest.mark.parametrize("nk", [8192, 16384])
def test_gemm_long_k_no_truncation_bias(nk):
    """U[0,1) data, long K: the tensor-core accumulate truncates, so without
    chunked promotion the result is biased low by ~(K/8)*2^-24 (1e-4 at K=16k).
    With 512-wide chunks promoted to fp32 registers the error stays ~1e-6 to 1e-5:
    the raw-hi split (round 2: the fp32 operand itself is hi, truncated to tf32 by
    the tensor core, lo = rna(x - trunc x)) measured 1.01e-5 at K = 8k
    under forced split-K 3 (round 1's rna-hi split stayed below 1e-5)."""
    r = P.check_gemm(256, 128, nk, 1.0, 0.0)
    assert r["err"] <= 2e-5, r["err"]
    assert abs(np.mean((r["g"] - r["r"]) / r["r"])) <= 1e-5  # no systematic bias


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_gemm_paper_variants(variant):
    _ok(P.check_gemm(130, 132, 200, variant=variant))


def test_listing8_equals_listing9_bitwise():
    """loop internalization preserves semantics; our SIMT
    twins keep the k order, so Listing 8 and Listing 9 agree bit for bit."""
    a = P.check_gemm(100, 96, 152, variant=0)["g"]
    b = P.check_gemm(100, 96, 152, variant=1)["g"]
    assert np.array_equal(a, b)


@pytest.mark.parametrize("dims", [(128, 128, 128, 128), (129, 132, 136, 124), (384, 260, 516, 260)])
def test_2mm(dims):
    _ok(P.check_2mm(*dims))


def test_2mm_chain_identity_P7():
    ni = nj = nk = nl = 256
    A, B, D = P.H(ni, nk, 1), P.H(nk, nj, 2), P.H(ni, nl, 4)
    C = np.eye(nj, dtype=np.float32)
    dD = P.dev(D)
    pb.pb_2mm(ni, nj, nk, nl, 1.5, 1.2, None, P.dev(A), P.dev(B), P.dev(C), dD)
    r = oracle.gemm(1.5, 1.2, D, A, B)
    s = oracle.gemm(1.5, 1.2, D, A, B, absmode=True)
    assert P.cerr(P.host(dD), r, s) <= P.TOL


@pytest.mark.parametrize("dims", [(128, 128, 128, 128, 128), (129, 132, 136, 124, 260), (260, 388, 132, 256, 300)])
def test_3mm(dims):
    _ok(P.check_3mm(*dims))


@pytest.mark.parametrize("n,m", [(128, 128), (132, 136), (260, 388), (512, 1028), (1000, 300)])
def test_syrk(n, m):
    _ok(P.check_syrk(n, m))


@pytest.mark.parametrize("n,m", [(128, 128), (132, 136), (388, 260), (516, 1024)])
def test_syr2k(n, m):
    _ok(P.check_syr2k(n, m))


def test_syr2k_equals_syrk_doubled_P12():
    n, m = 260, 300
    A = P.H(n, m, 1, mode=pbgen.INT8)
    C = P.H(n, n, 3, mode=pbgen.INT8 | pbgen.SYM)
    c1, c2 = P.dev(C), P.dev(C)
    dA = P.dev(A)
    pb.pb_syr2k(n, m, 1.5, 0.5, c1, dA, dA)
    pb.pb_syrk(n, m, 3.0, 0.5, c2, dA)
    assert np.array_equal(P.host(c1), P.host(c2))


def test_syrk_integer_bitwise_P1():
    n, m = 260, 1024
    A = P.H(n, m, 1, mode=pbgen.INT8)
    C = P.H(n, n, 3, mode=pbgen.INT8 | pbgen.SYM)
    dC = P.dev(C)
    pb.pb_syrk(n, m, 1.5, 0.5, dC, P.dev(A))
    assert np.array_equal(P.host(dC).astype(np.float64), oracle.syrk(1.5, 0.5, C, A))


@pytest.mark.parametrize("m,n", [(128, 128), (132, 137), (260, 517), (516, 2048)])
def test_covariance(m, n):
    _ok(P.check_covariance(m, n))


@pytest.mark.parametrize("m,n", [(128, 128), (132, 137), (260, 517), (516, 2048)])
def test_correlation(m, n):
    _ok(P.check_correlation(m, n))


def test_covariance_unstructured_ragged():
    _ok(P.check_covariance(388, 301, structured=False))


@pytest.mark.parametrize("m,n", [(132, 2049), (68, 3001)])
def test_cov_corr_long_columns_exact_mean_path(m, n):
    """n > 2048 rows: the exact-mean prep path (not the banded one)."""
    _ok(P.check_covariance(m, n))
    _ok(P.check_correlation(m, n))


@pytest.mark.parametrize("m,n", [(132, 255), (132, 257), (260, 1999), (64, 2048)])
def test_cov_corr_band_edges(m, n):
    """banded prep: ragged last band, single band, exactly 8 bands."""
    _ok(P.check_covariance(m, n))
    _ok(P.check_correlation(m, n))


# full-matrix syrk / syr2k (SYCL-Bench form): non-symmetric C, ragged sizes, split-K and tile configs
@pytest.mark.parametrize("n,m", [(4, 4), (132, 36), (300, 260), (1000, 516), (2048, 1028)])
@pytest.mark.parametrize("two", [False, True])
def test_syrk_full(n, m, two):
    _ok(P.check_syrk_full(n, m, two))


# ------------------------------------------------------------------ matrix-vector
# single-pass cluster kernel: n >= 16384 and A >= 96 MB (e.g. (2000, 32764), (1537, 16388), (300, 32768));
# else two passes (e.g. (6000, 4100): 98 MB of A with short rows)
@pytest.mark.parametrize("m,n", [(1, 4), (7, 8), (257, 516), (1000, 2052), (4096, 4096), (3001, 5000),
                                 (150, 32768), (5000, 1024), (148, 1028), (2000, 32764), (1537, 16388),
                                 (6000, 4100), (300, 32768)])
def test_atax(m, n):
    _ok(P.check_atax(m, n))


@pytest.mark.parametrize("m,n", [(4, 1), (8, 7), (516, 257), (2052, 1000), (4096, 4096), (5000, 3001)])
def test_bicg(m, n):
    _ok(P.check_bicg(m, n))


@pytest.mark.parametrize("n", [4, 8, 132, 516, 2052, 4096])
def test_mvt(n):
    _ok(P.check_mvt(n))


@pytest.mark.parametrize("n", [4, 8, 132, 516, 2052, 4096])
def test_gesummv(n):
    _ok(P.check_gesummv(n))


def test_atax_onepass_deterministic_and_tmp_optional():
    m, n = 1600, 16384  # single-pass path (n >= 16384, A >= 96 MB)
    A, x = P.dev(P.H(m, n, 1)), P.dev(P.H(1, n, 6)[0])
    ys = []
    for tmp in (None, torch.empty(m, device="cuda")):
        y = torch.empty(n, device="cuda")
        pb.pb_atax(m, n, A, x, y, tmp)
        ys.append(P.host(y))
    assert np.array_equal(ys[0], ys[1])


def test_matvec_deterministic_P32():
    n = 4096
    A, p, r = P.dev(P.H(n, n, 1)), P.dev(P.H(1, n, 6)[0]), P.dev(P.H(1, n, 7)[0])
    res = []
    for _ in range(2):
        s, q = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
        pb.pb_bicg(n, n, A, s, q, p, r)
        res.append((P.host(s), P.host(q)))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


# ------------------------------------------------------------------ ABI error behaviour
def test_abi_errors_leave_outputs_untouched():
    A = torch.ones(64, 64, device="cuda")
    B = torch.ones(64, 64, device="cuda")
    C = torch.full((64, 64), 3.0, device="cuda")
    with pytest.raises(pb.PBError) as e:  # alias: C overlaps A
        pb.pb_gemm(64, 64, 64, 1.0, 1.0, A, A, B)
    assert e.value.status == 3
    with pytest.raises(pb.PBError) as e:  # cols % 4
        pb.pb_gemm(64, 62, 64, 1.0, 1.0, C, A, B)
    assert e.value.status == 2
    with pytest.raises(pb.PBError) as e:  # misaligned pointer
        pb.pb_gemm(8, 8, 8, 1.0, 1.0, C.view(-1)[1:].data_ptr(), A, B)
    assert e.value.status == 2
    with pytest.raises(pb.PBError) as e:  # host pointer
        pb.pb_gemm(8, 8, 8, 1.0, 1.0, torch.ones(8, 8).data_ptr(), A, B)
    assert e.value.status == 1
    ws = torch.empty(256, dtype=torch.uint8, device="cuda")
    with pytest.raises(pb.PBError) as e:  # workspace too small
        pb.pb_gemm(64, 64, 64, 1.0, 1.0, C, A, B, ws=ws)
    assert e.value.status == 4
    assert bool((C == 3.0).all())


def test_row_sharded_pieces_match_full():
    """Host-side sharding math on one GPU: syrk_rows bands and matvec partials
    reassemble the single-call results (P33 on one device)."""
    n, m = 520, 300
    Ah, Ch = P.H(n, m, 1), P.H(n, n, 3, mode=pbgen.SYM)
    A = P.dev(Ah)
    parts = P.dev(Ch)
    for g in range(3):  # bands may run different tile configs: compare with the oracle
        r0, r1 = pb.pb_row_partition(n, 3, g, triangular=True, align=128)
        if r1 > r0:
            pb.pb_syrk_rows(n, m, r0, r1, 1.5, 1.2, parts[r0:r1], A)
    r = oracle.syrk(1.5, 1.2, Ch, Ah)
    s = oracle.syrk(1.5, 1.2, Ch, Ah, absmode=True)
    assert P.cerr(P.host(parts), r, s) <= P.TOL
    rows, cols = 1000, 1028
    A = P.dev(P.H(rows, cols, 1))
    v, w = P.dev(P.H(1, cols, 6)[0]), P.dev(P.H(1, rows, 7)[0])
    rd, cp = torch.empty(rows, device="cuda"), torch.empty(cols, device="cuda")
    pb.pb_matvec_partial(rows, cols, A, v, None, rd, w, None, cp)
    s, q = torch.empty(cols, device="cuda"), torch.empty(rows, device="cuda")
    pb.pb_bicg(cols, rows, A, s, q, v, w)
    assert np.array_equal(P.host(rd), P.host(q)) and np.array_equal(P.host(cp), P.host(s))


# ------------------------------------------------------------------ degenerate cases
def test_covariance_minimum_observations():
    """n = 2 observations (the minimum for float_n - 1), m = 4 variables."""
    _ok(P.check_covariance(4, 2, structured=False))
    _ok(P.check_correlation(4, 2, structured=False))


def test_correlation_single_observation_and_covariance_rejects_it():
    """n = 1: every stddev is 0 <= eps -> 1, so corr is the identity; covariance
    needs n >= 2 and must fail without touching its outputs."""
    data = P.dev(P.H(1, 8, 5))
    corr = torch.full((8, 8), 7.0, device="cuda")
    pb.pb_correlation(8, 1, 1.0, 0.1, data, corr, None, None)
    assert np.array_equal(P.host(corr), np.eye(8, dtype=np.float32))
    cov = torch.full((8, 8), 7.0, device="cuda")
    with pytest.raises(pb.PBError) as e:
        pb.pb_covariance(8, 1, 1.0, data, cov, None)
    assert e.value.status == 1 and bool((cov == 7.0).all())


@pytest.mark.parametrize("n", [3, 300, 2048, 2100])
def test_constant_data(n):
    """Every column constant (dyadic): covariance exactly 0, correlation exactly I
    (eps rule), means exact — on the banded (n <= 2048) and exact-mean paths."""
    m = 132
    h = np.tile((np.arange(m, dtype=np.float32) % 7) * 0.25, (n, 1))
    data = P.dev(h)
    cov, corr = torch.empty(m, m, device="cuda"), torch.empty(m, m, device="cuda")
    mean = torch.empty(m, device="cuda")
    pb.pb_covariance(m, n, float(n), data, cov, mean)
    pb.pb_correlation(m, n, float(n), 0.1, data, corr, None, None)
    assert np.array_equal(P.host(cov), np.zeros((m, m), np.float32))
    assert np.array_equal(P.host(corr), np.eye(m, dtype=np.float32))
    assert np.array_equal(P.host(mean), h[0])


def test_gemm_single_row_long_k_tensor_path():
    """M = 1 (one ragged row in a 128-row tile), N = 8, K = 262144: the tensor-core
    path (above the small-problem threshold) with split-K over a very long K."""
    _ok(P.check_gemm(1, 8, 262144))


# ------------------------------------------------------------------ P1 on the chains and the matvec family
def test_2mm_3mm_integer_bitwise_P1():
    """Values in {0..7}, dyadic alpha/beta, sizes keeping every partial sum < 2^24:
    the 3xTF32 chain is exact (the intermediate's hi/lo split is exact too), so
    tmp/D and E/F/G equal the oracle bit for bit."""
    I8 = pbgen.INT8
    ni, nj, nk, nl = 300, 32, 64, 260
    A, B, C, D = P.H(ni, nk, 1, I8), P.H(nk, nj, 2, I8), P.H(nj, nl, 3, I8), P.H(ni, nl, 4, I8)
    dtmp, dD = torch.empty(ni, nj, device="cuda"), P.dev(D)
    pb.pb_2mm(ni, nj, nk, nl, 1.5, 0.5, dtmp, P.dev(A), P.dev(B), P.dev(C), dD)
    t_r, D_r = oracle.mm2(1.5, 0.5, A, B, C, D)
    assert np.array_equal(P.host(dtmp).astype(np.float64), t_r)
    assert np.array_equal(P.host(dD).astype(np.float64), D_r)
    ni, nj, nk, nl, nm = 260, 16, 8, 132, 8
    A, B, C, D = P.H(ni, nk, 1, I8), P.H(nk, nj, 2, I8), P.H(nj, nm, 3, I8), P.H(nm, nl, 4, I8)
    dE, dF, dG = (torch.empty(*sh, device="cuda") for sh in ((ni, nj), (nj, nl), (ni, nl)))
    pb.pb_3mm(ni, nj, nk, nl, nm, dE, P.dev(A), P.dev(B), dF, P.dev(C), P.dev(D), dG)
    for g, r in zip((dE, dF, dG), oracle.mm3(A, B, C, D)):
        assert np.array_equal(P.host(g).astype(np.float64), r)


def test_matvec_integer_bitwise_P1():
    """bicg / mvt / gesummv with values in {0..7} at n = 2048 (sums < 2^24, dyadic
    alpha/beta): exact, so bit-for-bit equal to the oracle despite different
    reduction orders; mvt with a symmetric A and y_1 = y_2 then also gives
    x1' - x1 == x2' - x2 exactly (P28 on the GPU)."""
    I8 = pbgen.INT8
    n = 2048
    A = P.H(n, n, 1, I8)
    p, r = P.H(1, n, 6, I8)[0], P.H(1, n, 7, I8)[0]
    s, q = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    pb.pb_bicg(n, n, P.dev(A), s, q, P.dev(p), P.dev(r))
    s_r, q_r = oracle.bicg(A, p, r)
    assert np.array_equal(P.host(s).astype(np.float64), s_r) and np.array_equal(P.host(q).astype(np.float64), q_r)
    B = P.H(n, n, 2, I8)
    y, t = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    pb.pb_gesummv(n, 1.5, 0.5, P.dev(A), P.dev(B), t, P.dev(p), y)
    t_r, y_r = oracle.gesummv(1.5, 0.5, A, B, p)
    assert np.array_equal(P.host(t).astype(np.float64), t_r) and np.array_equal(P.host(y).astype(np.float64), y_r)
    As = P.H(n, n, 1, I8 | pbgen.SYM)
    x1, x2 = P.H(1, n, 8, I8)[0], P.H(1, n, 9, I8)[0]
    d1, d2 = P.dev(x1), P.dev(x2)
    pb.pb_mvt(n, d1, d2, P.dev(p), P.dev(p), P.dev(As))
    o1, o2 = oracle.mvt(x1, x2, p, p, As)
    g1, g2 = P.host(d1).astype(np.float64), P.host(d2).astype(np.float64)
    assert np.array_equal(g1, o1) and np.array_equal(g2, o2)
    assert np.array_equal(g1 - x1, g2 - x2)


@pytest.mark.parametrize("two", [False, True])
def test_syrk_syr2k_beta0_nan_not_read(two):
    """beta == 0: C's lower triangle is write-only (include/pb.h BLAS convention), so NaN
    there must not propagate; the strict upper triangle is untouched (NaN stays NaN)."""
    n, m = 260, 132
    A, B = P.H(n, m, 1), P.H(n, m, 2)
    C = np.full((n, n), np.nan, dtype=np.float32)
    dC = P.dev(C)
    if two:
        pb.pb_syr2k(n, m, 1.5, 0.0, dC, P.dev(A), P.dev(B))
        r = oracle.syr2k(1.5, 0.0, np.zeros_like(C), A, B)
        s = oracle.syr2k(1.5, 0.0, np.zeros_like(C), A, B, absmode=True)
    else:
        pb.pb_syrk(n, m, 1.5, 0.0, dC, P.dev(A))
        r = oracle.syrk(1.5, 0.0, np.zeros_like(C), A)
        s = oracle.syrk(1.5, 0.0, np.zeros_like(C), A, absmode=True)
    g = P.host(dC)
    low = np.tril(np.ones((n, n), bool))
    assert P.cerr(g[low], r[low], s[low]) <= P.TOL
    assert np.all(np.isnan(g[~low]))


def test_2mm_beta0_nan_not_read():
    ni, nj, nk, nl = 132, 136, 260, 128
    A, B, C = P.H(ni, nk, 1), P.H(nk, nj, 2), P.H(nj, nl, 3)
    dD = P.dev(np.full((ni, nl), np.nan, dtype=np.float32))
    pb.pb_2mm(ni, nj, nk, nl, 1.5, 0.0, None, P.dev(A), P.dev(B), P.dev(C), dD)
    (_, Dr), (_, Ds) = (oracle.mm2(1.5, 0.0, A, B, C, np.zeros((ni, nl), np.float32), absmode=a) for a in (False, True))
    assert P.cerr(P.host(dD), Dr, Ds) <= P.TOL


@pytest.mark.parametrize("m,n", [(1024, 4096), (3072, 4096)])
def test_cov_corr_exact_mean_path_workspace_bound(m, n):
    """n > 2048 (exact-mean prep) with m large enough that the Gram plan splits K through
    the partial buffer (the split-K area was once sized for the other
    plan): the call gets a workspace of exactly pb_workspace_size bytes followed by a
    sentinel region, which must come back untouched; results against the oracle."""
    import oracle
    data = P.H(n, m, P.S["data"])
    for k in ("covariance", "correlation"):
        need = pb.workspace_size(k, (m, n))
        buf = torch.full((need + (1 << 20),), 0xAB, dtype=torch.uint8, device="cuda")
        ws = buf[:need]
        out = torch.empty(m, m, device="cuda")
        if k == "covariance":
            pb.pb_covariance(m, n, float(n), P.dev(data), out, None, ws=ws)
            r, s = oracle.covariance(float(n), data)[0], oracle.covariance(float(n), data, absmode=True)[0]
        else:
            pb.pb_correlation(m, n, float(n), 0.1, P.dev(data), out, None, None, ws=ws)
            r, s = oracle.correlation(float(n), 0.1, data)[0], oracle.correlation(float(n), 0.1, data, absmode=True)[0]
        assert bool((P.host(buf[need:]) == 0xAB).all()), f"{k}: workspace overrun"
        assert P.cerr(P.host(out), r, s) <= P.TOL, k
