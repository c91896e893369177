"""Race evidence by repetition (SURVEY §5 race detection; VERDICT r01 missing #6).

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset; see
profiles/r02_sanitizer_refused.log), so the hand-synchronised kernels are checked the way a
race shows up without it: bitwise reproducibility over many repetitions, with the launch order
and L2 state perturbed between repetitions (a 256 MB scrub of L2 and a busy kernel on a side
stream), and against the oracle where the result is exactly defined.
  - k_chol_dag       cross-CTA tile flags (release/acquire) and per-tile update counters
  - trsv_ws          per-block mbarriers + st.async DSMEM broadcast inside 8-CTA clusters
  - k_qr_step_v4     per-row team barrier of the in-place update (round 2's race fix)
  - k_gram_fused     ring hand-off counters across CTAs (opt-in path)
  - k_gram_tc2       the 2-deep TMEM ring, coalesced fp64 flushes through shared memory
  - k_wpcg_step_coop grid barriers + the fused partial reduction
"""
import os

import numpy as np
import pytest
import torch

import tlsgen
from oracle import rqi

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

REPS = int(os.environ.get("TLS_STRESS_REPS", "12"))


@pytest.fixture(scope="module")
def T():
    from paper_2305_19028_b200 import tlsrqi
    tlsrqi.lib()
    return tlsrqi


def _perturb(i):
    """Scrub L2 (write 256 MB) and keep a side stream busy so that CTA scheduling and cache
    state differ from repetition to repetition."""
    buf = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
    buf.fill_(float(i))
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        x = torch.randn(2048, 2048, device="cuda")
        for _ in range(i % 3):
            x = x @ x
    return side, x


def _bits(t):
    return t.detach().cpu().numpy().view(np.uint64).copy()


@pytest.mark.parametrize("n,u_f", [(1000, "fp16"), (2048, "bf16")])
def test_cholesky_and_solves_bitwise_reproducible(T, n, u_f):
    P = tlsgen.dense_problem(4 * n, n, 1e2, 1e-3, 3, twin=True, device="cuda", keep_factors=False)
    M = T.matrix(P.A)
    ws = T.workspace(M)
    ref_R = ref_x = None
    for i in range(REPS):
        side, _ = _perturb(i)
        rc, R, _ = T.tls_factor_precond(M, u_f, ws=ws)
        rc2, x, sig, info = T.tls_rqi_pcgtls(M, P.b, R, ws=ws)
        torch.cuda.synchronize()
        side.synchronize()
        Rt, d, nrm = T.tls_precond_export(R)
        if ref_R is None:
            ref_R, ref_x, ref_info = Rt, _bits(x), info
        assert np.array_equal(Rt, ref_R), f"R~ differs at repetition {i}"
        assert np.array_equal(_bits(x), ref_x), f"x differs at repetition {i}"
        assert info["pcg_iters"] == ref_info["pcg_iters"]


def test_explicit_inverse_step_bitwise_reproducible(T):
    P = tlsgen.config("cfg2w")
    A = torch.as_tensor(P.A, device="cuda")
    b = torch.as_tensor(P.b, device="cuda")
    M = T.matrix(A)
    rc, R, _ = T.tls_factor_precond(M, "bf16")
    o = T.tls_rqi_opts_default(precond_apply=2)
    ref = None
    for i in range(REPS):
        side, _ = _perturb(i)
        rc, x, sig, info = T.tls_rqi_pcgtls(M, b, R, opts=o)
        torch.cuda.synchronize()
        side.synchronize()
        if ref is None:
            ref = _bits(x)
        assert np.array_equal(_bits(x), ref)


@pytest.mark.parametrize("m,n,fmt", [(1100, 530, "fp16"), (3000, 700, "bf16")])
def test_qr_bitwise_equal_to_oracle_every_repetition(T, m, n, fmt):
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n)) * np.exp2(rng.integers(-4, 5, n))[None, :]
    pc = rqi.factor_precond_qr(A, fmt)
    At = torch.as_tensor(A, device="cuda")
    M = T.matrix(At)
    for i in range(max(3, REPS // 3)):
        side, _ = _perturb(i)
        rc, R, _ = T.tls_factor_precond_qr(M, fmt)
        torch.cuda.synchronize()
        side.synchronize()
        Rt, d, nrm = T.tls_precond_export(R)
        assert np.array_equal(Rt, pc.Rt), f"QR R~ differs from the oracle at repetition {i}"


def test_fused_gram_bitwise_reproducible(T, monkeypatch):
    monkeypatch.setenv("TLS_GRAM_FUSED", "1")
    m, n = 200000, 1024
    A = torch.randn((m, n), dtype=torch.float64, device="cuda")
    M = T.matrix(A)
    ws = T.workspace(M)
    d = torch.full((n,), 8.0, dtype=torch.float64, device="cuda")
    ref = None
    for i in range(max(3, REPS // 2)):
        side, _ = _perturb(i)
        rc, G = T.tls_gram(M, "fp16", d, 64, ws=ws)
        torch.cuda.synchronize()
        side.synchronize()
        assert rc == 0
        if ref is None:
            ref = _bits(G)
        assert np.array_equal(_bits(G), ref)
    monkeypatch.setenv("TLS_GRAM_FUSED", "0")
    monkeypatch.setenv("TLS_GRAM_SEGS", "1")          # the unsegmented two-kernel path: same chunking
    monkeypatch.setenv("TLS_GRAM_TC", "128")          # and the same 128 x 128 tiles and splits
    rc, G0 = T.tls_gram(M, "fp16", d, 64, ws=ws)
    assert np.array_equal(_bits(G0), ref)            # and equal to the two-kernel path


@pytest.mark.parametrize("segs", ["8", "1"])
def test_gram_tc2_bitwise_reproducible(T, monkeypatch, segs):
    """The default dense Gram (k_gram_tc2, 128 x 256 blocks, rounding overlapped by segments):
    G bit-identical over repetitions."""
    monkeypatch.setenv("TLS_GRAM_SEGS", segs)
    m, n = 300000, 1000                                 # n > 896: the 128 x 256 kernel
    A = torch.randn((m, n), dtype=torch.float64, device="cuda")
    M = T.matrix(A)
    ws = T.workspace(M)
    d = torch.full((n,), 8.0, dtype=torch.float64, device="cuda")
    ref = None
    for i in range(max(3, REPS // 2)):
        side, _ = _perturb(i)
        rc, G = T.tls_gram(M, "bf16", d, 64, ws=ws)
        torch.cuda.synchronize()
        side.synchronize()
        assert rc == 0
        if ref is None:
            ref = _bits(G)
        assert np.array_equal(_bits(G), ref)


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_gram_fused2_equals_two_kernel(T, monkeypatch, fmt):
    """The opt-in split-role fused Gram (k_gram_fused2: converter CTAs write fl_uf(A D^-1) into an
    L2 ring that the SYRK CTAs read) gives G bit-identical to the two-kernel path (k_round_scaled
    + k_gram_tc2) run with the same 3 splits and one segment, over repetitions."""
    m, n = 300001, 1000
    A = T.dense_operand(torch.randn((m, n), dtype=torch.float64, device="cuda"))
    M = T.matrix(A)
    ws = T.workspace(M)
    d = torch.exp2(torch.randint(-3, 4, (n,), device="cuda").double())
    monkeypatch.setenv("TLS_GRAM_NSPLIT", "3")
    monkeypatch.setenv("TLS_GRAM_FUSED", "0")
    monkeypatch.setenv("TLS_GRAM_SEGS", "1")
    rc, G0 = T.tls_gram(M, fmt, d, 64, ws=ws)
    assert rc == 0
    ref = _bits(G0)
    monkeypatch.setenv("TLS_GRAM_FUSED", "2")
    for i in range(3):
        side, _ = _perturb(i)
        rc, G = T.tls_gram(M, fmt, d, 64, ws=ws)
        torch.cuda.synchronize()
        side.synchronize()
        assert rc == 0
        assert np.array_equal(_bits(G), ref)


@pytest.mark.parametrize("segs", ["1", "8"])
def test_gram_multicast_clusters_bit_identical(T, monkeypatch, segs):
    """k_gram_tc2 with 2-CTA clusters sharing the B panel by TMA multicast (opt-in TLS_GRAM_MC=1,
    empty barriers of count 2 fed by multicast commits) gives G bit-identical to the
    unclustered kernel, over repetitions."""
    monkeypatch.setenv("TLS_GRAM_SEGS", segs)
    m, n = 300001, 1000
    A = T.dense_operand(torch.randn((m, n), dtype=torch.float64, device="cuda"))
    M = T.matrix(A)
    ws = T.workspace(M)
    d = torch.exp2(torch.randint(-3, 4, (n,), device="cuda").double())
    monkeypatch.setenv("TLS_GRAM_MC", "0")
    rc, G0 = T.tls_gram(M, "fp16", d, 64, ws=ws)
    ref = _bits(G0)
    monkeypatch.setenv("TLS_GRAM_MC", "1")
    for i in range(3):
        side, _ = _perturb(i)
        rc, G = T.tls_gram(M, "fp16", d, 64, ws=ws)
        torch.cuda.synchronize()
        side.synchronize()
        assert rc == 0 and np.array_equal(_bits(G), ref)


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
@pytest.mark.parametrize("m,n", [(300001, 1000), (20001, 257), (70001, 2000), (40001, 1030)])
def test_gram_rounding_forms_bit_identical(T, monkeypatch, fmt, m, n):
    """The Gram's rounding pass fl_uf(A D^-1) in its three forms (TLS_ROUND=1: one row in flight
    per thread; default: two rows; 3: rows staged in shared memory by the bulk-copy engine, even n,
    one or two column chunks with a short second chunk) gives bit-identical G, alone and overlapped with the segmented
    SYRK, incl. odd n (a last column without a pair partner) and ragged m; and the same range
    flag when an entry overflows u_f."""
    A = T.dense_operand(torch.randn((m, n), dtype=torch.float64, device="cuda"))
    M = T.matrix(A)
    ws = T.workspace(M)
    d = torch.full((n,), 8.0, dtype=torch.float64, device="cuda")
    for segs in ("8", "1"):
        monkeypatch.setenv("TLS_GRAM_SEGS", segs)
        ref = None
        for rv in ("1", "2", "3"):
            monkeypatch.setenv("TLS_ROUND", rv)
            rc, G = T.tls_gram(M, fmt, d, 64, ws=ws)
            torch.cuda.synchronize()
            assert rc == 0
            if ref is None:
                ref = _bits(G)
            assert np.array_equal(_bits(G), ref), (segs, rv)
    if fmt == "fp16":                                   # one entry beyond fp16's range after scaling
        A[m // 2, n - 1] = 1e6
        rcs = set()
        for rv in ("1", "2", "3"):
            monkeypatch.setenv("TLS_ROUND", rv)
            rc, _ = T.tls_gram(M, fmt, d, 64, ws=ws)
            torch.cuda.synchronize()
            rcs.add(rc)
        assert len(rcs) == 1 and rcs.pop() != 0
