"""Kernel-level numerics of libfdmd on the GPU against numpy fp64 (the
oracle for plain linear algebra). FP64 kernels must match to ~1e-13
relative; fp32 outputs to fp32 rounding."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_05339_b200 import device
    return device


def _tall_from(dv, M, layout, dtype):
    n, k = M.shape
    T = dv.alloc_tall(n, k, dtype, layout, zero=True)
    src = torch.as_tensor(M, dtype=dtype)
    if layout == "row":
        T.buf[:n, :k].copy_(src)
    else:
        T.buf[:k, :n].copy_(src.t())
    return T


@pytest.mark.parametrize("a_layout", ["row", "col"])
@pytest.mark.parametrize("a_dtype", ["f32", "f64"])
@pytest.mark.parametrize("c_layout,c_dtype", [("row", "f64"), ("col", "f64"), ("col", "f32"), ("row", "f32")])
@pytest.mark.parametrize("shape", [(1000, 37, 20), (4099, 201, 210), (130, 16, 130), (64, 5, 3), (7, 201, 160)])
def test_tall_gemm(dv, a_layout, a_dtype, c_layout, c_dtype, shape):
    n, K, N = shape
    rng = np.random.default_rng(n + K + N)
    A = rng.standard_normal((n, K))
    ta = torch.float32 if a_dtype == "f32" else torch.float64
    if a_dtype == "f32":
        A = A.astype(np.float32).astype(np.float64)
    B = rng.standard_normal((K, N))
    At = _tall_from(dv, A, a_layout, ta)
    tc = torch.float32 if c_dtype == "f32" else torch.float64
    C = dv.alloc_tall(n, N, tc, c_layout)
    dv.get_ops().tall_gemm(At, torch.as_tensor(B, device="cuda"), C)
    got = C.view().double().cpu().numpy()
    want = A @ B
    tol = 1e-6 if c_dtype == "f32" else 1e-12
    assert np.abs(got - want).max() <= tol * max(np.abs(want).max(), 1.0)


def test_tall_gemm_pair_stats(dv):
    rng = np.random.default_rng(3)
    n, K, U = 5000, 31, 9
    A = rng.standard_normal((n, K))
    B = rng.standard_normal((K, 2 * U))
    At = _tall_from(dv, A, "row", torch.float64)
    C = dv.alloc_tall(n, 2 * U, torch.float64, "col")
    st = dv.get_ops().tall_gemm(At, torch.as_tensor(B, device="cuda"), C, stats=True, row_offset=11).cpu().numpy()
    P = A @ B
    mag = P[:, 0::2] ** 2 + P[:, 1::2] ** 2
    np.testing.assert_allclose(st[:, 0], mag.sum(0), rtol=1e-12)
    np.testing.assert_allclose(st[:, 1], mag.max(0), rtol=1e-13)
    np.testing.assert_array_equal(st[:, 2].astype(np.int64), mag.argmax(0) + 11)
    # stats-only pass (no output) gives the same statistics
    st2 = dv.get_ops().tall_gemm(At, torch.as_tensor(B, device="cuda"), None, stats=True, row_offset=11).cpu().numpy()
    np.testing.assert_array_equal(st, st2)


def test_tall_gemm_ring_variant_matches(dv):
    """The cp.async-ring kernel (FDMD_TG_IMPL=cpasync, used when TMA cannot
    describe the operand) gives the same results as the default TMA kernel."""
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2502_05339_b200 import device as dv
rng = np.random.default_rng(1)
for (n, K, N, lay) in [(5000, 201, 200, 'row'), (777, 37, 64, 'col'), (4099, 200, 128, 'row')]:
    A = rng.standard_normal((n, K)).astype(np.float32).astype(np.float64)
    T = dv.alloc_tall(n, K, torch.float32, lay, zero=True)
    (T.buf[:n, :K] if lay == 'row' else T.buf[:K, :n]).copy_(torch.as_tensor(A if lay == 'row' else A.T))
    B = rng.standard_normal((K, N))
    C = dv.alloc_tall(n, N, torch.float64, 'row')
    dv.get_ops().tall_gemm(T, torch.as_tensor(B, device='cuda'), C)
    err = np.abs(C.view().cpu().numpy() - A @ B).max() / np.abs(A @ B).max()
    assert err < 1e-12, err
print('ok')
"""
    env = dict(os.environ, FDMD_TG_IMPL="cpasync")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("upper", [False, True])
@pytest.mark.parametrize("l", [200, 37, 160])
def test_tall_gemm_inplace(dv, upper, l):
    rng = np.random.default_rng(4 + l)
    n = 3000
    Y = rng.standard_normal((n, l))
    R = np.triu(rng.standard_normal((l, l))) + 5 * np.eye(l)
    Yt = _tall_from(dv, Y, "row", torch.float64)
    dv.get_ops().tall_gemm(Yt, torch.as_tensor(R, device="cuda"), Yt, upper=upper)
    np.testing.assert_allclose(Yt.view().cpu().numpy(), Y @ R, rtol=0, atol=1e-11 * np.abs(Y @ R).max())


@pytest.mark.parametrize("K", [200, 13, 64, 71])
def test_tall_gram_symmetric_shapes(dv, K):
    rng = np.random.default_rng(K)
    n = 5003
    Y = rng.standard_normal((n, K))
    for layout in ("row", "col"):
        Yt = _tall_from(dv, Y, layout, torch.float64)
        G = dv.get_ops().tall_gram(Yt, Yt, symmetric=True).cpu().numpy()
        np.testing.assert_allclose(G, Y.T @ Y, rtol=0, atol=1e-12 * np.abs(Y.T @ Y).max())


@pytest.mark.parametrize("la,lb", [("row", "row"), ("col", "row"), ("row", "col"), ("col", "col")])
@pytest.mark.parametrize("da,db", [("f32", "f32"), ("f64", "f32"), ("f64", "f64")])
@pytest.mark.parametrize("shape", [(10000, 200, 201), (333, 30, 101), (17, 5, 3), (70000, 64, 64)])
def test_tall_gram(dv, la, lb, da, db, shape):
    n, K1, K2 = shape
    rng = np.random.default_rng(n + K1)
    A = rng.standard_normal((n, K1))
    B = rng.standard_normal((n, K2))
    if da == "f32":
        A = A.astype(np.float32).astype(np.float64)
    if db == "f32":
        B = B.astype(np.float32).astype(np.float64)
    At = _tall_from(dv, A, la, torch.float32 if da == "f32" else torch.float64)
    Bt = _tall_from(dv, B, lb, torch.float32 if db == "f32" else torch.float64)
    G = dv.get_ops().tall_gram(At, Bt).cpu().numpy()
    want = A.T @ B
    assert np.abs(G - want).max() <= 1e-12 * np.abs(want).max() * max(1, np.sqrt(n) / 100)


@pytest.mark.parametrize("K1,K2,sym", [(200, 200, True), (256, 256, True), (400, 400, True), (150, 150, True),
                                       (8, 8, True), (1, 1, True), (200, 201, False), (201, 200, False),
                                       (40, 300, False), (400, 401, False), (3, 5, False)])
@pytest.mark.parametrize("n", [1, 16, 17, 40001])
@pytest.mark.parametrize("da,db", [("f64", "f64"), ("f32", "f64"), ("f64", "f32")])
def test_tall_gram_panel_shapes(dv, K1, K2, sym, n, da, db):
    """Row-major operands take the panel kernel (whole output per CTA
    partition); K past 8 partitions falls back to the tiled kernel."""
    if sym and da != db:
        pytest.skip("symmetric Gram has one operand")
    rng = np.random.default_rng(K1 * 1000 + K2 + n)
    tA = torch.float32 if da == "f32" else torch.float64
    tB = torch.float32 if db == "f32" else torch.float64
    A = rng.standard_normal((n, K1))
    if da == "f32":
        A = A.astype(np.float32).astype(np.float64)
    At = _tall_from(dv, A, "row", tA)
    if sym:
        G = dv.get_ops().tall_gram(At, At, symmetric=True).cpu().numpy()
        want = A.T @ A
        assert np.array_equal(G, G.T)
    else:
        B = rng.standard_normal((n, K2))
        if db == "f32":
            B = B.astype(np.float32).astype(np.float64)
        Bt = _tall_from(dv, B, "row", tB)
        G = dv.get_ops().tall_gram(At, Bt).cpu().numpy()
        want = A.T @ B
    assert np.abs(G - want).max() <= 1e-12 * max(np.abs(want).max(), 1e-300) * max(1, np.sqrt(n) / 100)


def test_tall_gram_panel_matches_tiled_kernel(tmp_path):
    """The panel and the 64 x TN tiled Gram agree (FDMD_GRAM_IMPL=tile)."""
    code = (
        "import numpy as np, torch, sys\n"
        "sys.path.insert(0, '.')\n"
        "from paper_2502_05339_b200 import device as dv\n"
        "rng = np.random.default_rng(3)\n"
        "out = {}\n"
        "Y = torch.as_tensor(rng.standard_normal((300001, 200)), device='cuda')\n"
        "S = torch.as_tensor(rng.standard_normal((300001, 201)), device='cuda', dtype=torch.float32)\n"
        "from paper_2502_05339_b200.linalg import as_tall\n"
        "Yt, St = as_tall(Y), as_tall(S)\n"
        "ops = dv.get_ops()\n"
        "out['sym'] = ops.tall_gram(Yt, Yt, symmetric=True).cpu().numpy()\n"
        "out['qts'] = ops.tall_gram(Yt, St).cpu().numpy()\n"
        "out['stq'] = ops.tall_gram(St, Yt).cpu().numpy()\n"
        f"np.savez(sys.argv[1], **out)\n")
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for impl in ("panel", "tile"):
        f = tmp_path / f"{impl}.npz"
        env = dict(os.environ, FDMD_GRAM_IMPL=impl)
        subprocess.run([sys.executable, "-c", code, str(f)], cwd=root, env=env, check=True, timeout=300)
        res[impl] = np.load(f)
    for k in ("sym", "qts", "stq"):
        a, b = res["panel"][k], res["tile"][k]
        assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max(), k


def test_tall_gram_symmetric_deterministic(dv):
    rng = np.random.default_rng(5)
    Y = rng.standard_normal((200000, 210))
    Yt = _tall_from(dv, Y, "row", torch.float64)
    G1 = dv.get_ops().tall_gram(Yt, Yt, symmetric=True).cpu().numpy()
    G2 = dv.get_ops().tall_gram(Yt, Yt, symmetric=True).cpu().numpy()
    assert np.array_equal(G1, G2)
    assert np.array_equal(G1, G1.T)
    np.testing.assert_allclose(G1, Y.T @ Y, rtol=0, atol=1e-12 * np.abs(Y.T @ Y).max())


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("B", [1, 2, 3, 8, 13, 32, 45])
@pytest.mark.parametrize("n,r", [(10007, 150), (64, 7), (100003, 200)])
def test_decode(dv, dtype, B, n, r):
    rng = np.random.default_rng(B * 7 + r)
    D = rng.standard_normal((n, r))
    C = rng.standard_normal((r, B))
    td = torch.float32 if dtype == "f32" else torch.float64
    if dtype == "f32":
        D = D.astype(np.float32).astype(np.float64)
        C = C.astype(np.float32).astype(np.float64)
    Dt = _tall_from(dv, D, "col", td)
    out = dv.get_ops().decode(Dt, torch.as_tensor(C, device="cuda", dtype=td)).double().cpu().numpy()
    want = (D @ C).T
    tol = 2e-6 if dtype == "f32" else 1e-13
    assert np.linalg.norm(out - want) <= tol * np.linalg.norm(want)


@pytest.mark.parametrize("n,r,B", [(100003, 200, 32), (5000, 150, 128), (70000, 200, 300), (257, 7, 16),
                                   (100000, 256, 129), (70001, 200, 512), (30011, 150, 1024), (5000, 64, 640),
                                   (300, 200, 384), (40000, 200, 2100)])
def test_tc_decode_fp16_split(dv, n, r, B):
    """tcgen05 2-way FP16 split reconstruction: FP32-accurate (rel-L2 per frame).
    B > 128 runs as clusters of 2/4/8 CTAs sharing basis chunks by TMA
    multicast (ragged cluster tails: B = 300, 640, 2100)."""
    rng = np.random.default_rng(n + r + B)
    U = np.linalg.qr(rng.standard_normal((n, r)))[0] if n >= r else rng.standard_normal((n, r))
    U = U.astype(np.float32).astype(np.float64)
    C = rng.standard_normal((r, B)) * np.exp(rng.uniform(-8, 3, B))[None, :]   # frames of very different scale
    Ut = _tall_from(dv, U, "col", torch.float32)
    ops = dv.get_ops()
    tcb = ops.tc_basis(Ut)
    out = ops.tc_decode(tcb, torch.as_tensor(C, device="cuda")).double().cpu().numpy()
    want = (U @ C.astype(np.float32).astype(np.float64)).T
    err = np.linalg.norm(out - want, axis=1) / np.linalg.norm(want, axis=1)
    assert err.max() <= 2e-6, err.max()


@pytest.mark.parametrize("n,K,k", [(100003, 200, 200), (70001, 160, 150), (5000, 64, 37), (3000, 256, 256)])
def test_tc_decode_planes_lift(dv, n, K, k):
    """The lift U = Q M written straight into fp16 hi/lo planes
    (fdmd_tc_decode_planes): the planes hold U to FP32 accuracy, columns past k
    are zero, and reconstructing frames from them equals U @ C."""
    rng = np.random.default_rng(n + K + k)
    Q = np.linalg.qr(rng.standard_normal((n, K)))[0] if n >= K else rng.standard_normal((n, K)) / np.sqrt(n)
    M = np.linalg.qr(rng.standard_normal((K, K)))[0][:, :k]          # U = Q M: orthonormal columns, |U| <= 1
    ops = dv.get_ops()
    Qt = _tall_from(dv, Q, "row", torch.float64)
    qt = ops.tc_rows(Qt, bound=2.0)
    pl = ops.tc_decode_planes(qt, torch.as_tensor(M, device="cuda"), bound=2.0)
    U = (pl["uh"].double() + pl["ul"].double()).cpu().numpy() / pl["su"]
    want = Q @ M
    assert pl["ldu"] % 8 == 0 and np.all(U[:, k:] == 0.0)
    err = np.linalg.norm(U[:, :k] - want, axis=0) / np.linalg.norm(want, axis=0)
    assert err.max() <= 2e-6, err.max()
    C = rng.standard_normal((k, 40))
    fr = ops.tc_decode(pl, torch.as_tensor(C, device="cuda")).double().cpu().numpy()
    wf = (want @ C.astype(np.float32).astype(np.float64)).T
    assert (np.linalg.norm(fr - wf, axis=1) / np.linalg.norm(wf, axis=1)).max() <= 4e-6


@pytest.mark.parametrize("n,m,k,dt", [(100003, 201, 200, torch.float32), (70001, 161, 150, torch.float32),
                                       (5000, 40, 37, torch.float64), (3001, 256, 256, torch.float32)])
def test_tall_gemm_planes_lift(dv, n, m, k, dt):
    """The lift U = S Umap on FP64 DMMA written straight into fp16 hi/lo planes
    (fdmd_tall_gemm_planes, the projection-from-Gram route): S is an
    ill-conditioned snapshot-like matrix and Umap = (its R factor)^-1 times an
    orthogonal map, so U has orthonormal columns only through cancellation
    (~cond(S) = 1e4) — the planes still hold U to FP32 accuracy, padding
    columns are zero, and tc_decode from them reproduces U @ C."""
    rng = np.random.default_rng(n + m + k)
    sv = np.logspace(0, -4, m)
    S = (np.linalg.qr(rng.standard_normal((n, m)))[0] * sv) @ np.linalg.qr(rng.standard_normal((m, m)))[0]
    S = S.astype(np.float32 if dt == torch.float32 else np.float64)
    Sd = S.astype(np.float64)
    R = np.linalg.qr(Sd)[1]
    Umap = np.linalg.solve(R, np.linalg.qr(rng.standard_normal((m, m)))[0][:, :k])
    want = Sd @ Umap
    ops = dv.get_ops()
    St = _tall_from(dv, S, "row", dt)
    pl = ops.tall_gemm_planes(St, torch.as_tensor(Umap, device="cuda"), bound=2.0)
    U = (pl["uh"].double() + pl["ul"].double()).cpu().numpy() / pl["su"]
    assert pl["ldu"] % 8 == 0 and np.all(U[:, k:] == 0.0)
    err = np.linalg.norm(U[:, :k] - want, axis=0) / np.linalg.norm(want, axis=0)
    assert err.max() <= 2e-6, err.max()
    C = rng.standard_normal((k, 40))
    fr = ops.tc_decode(pl, torch.as_tensor(C, device="cuda")).double().cpu().numpy()
    wf = (want @ C.astype(np.float32).astype(np.float64)).T
    assert (np.linalg.norm(fr - wf, axis=1) / np.linalg.norm(wf, axis=1)).max() <= 4e-6


@pytest.mark.parametrize("n,m,dt", [(1000003, 201, torch.float32), (70001, 41, torch.float64), (5, 3, torch.float32)])
def test_tall_tdot_border(dv, n, m, dt):
    """fdmd_tall_tdot: the border X^T s_m of the snapshot Gram (last column of
    a row-major padded S against the first T = m - 1), fp64 accumulation,
    bitwise repeatable, and beta accumulation for the streamed upload."""
    rng = np.random.default_rng(n + m)
    S = rng.standard_normal((n, m)).astype(np.float32 if dt == torch.float32 else np.float64)
    Sd = S.astype(np.float64)
    want = Sd[:, : m - 1].T @ Sd[:, m - 1]
    St = _tall_from(dv, S, "row", dt)
    ops = dv.get_ops()
    y = ops.tall_tdot(St, m - 1, m - 1)
    np.testing.assert_allclose(y.cpu().numpy(), want, rtol=1e-12, atol=1e-12 * np.abs(Sd).max() ** 2 * n)
    assert torch.equal(y, ops.tall_tdot(St, m - 1, m - 1))
    acc = y.clone()
    ops.tall_tdot(St, m - 1, m - 1, out=acc, beta=1.0)
    np.testing.assert_allclose(acc.cpu().numpy(), 2 * want, rtol=1e-12, atol=1e-12 * np.abs(Sd).max() ** 2 * n)


@pytest.mark.parametrize("n,K,dt", [(300007, 200, torch.float32), (70001, 200, torch.float64),
                                    (50021, 150, torch.float32), (4099, 20, torch.float64),
                                    (65536, 100, torch.float32), (33333, 256, torch.float32),
                                    (20011, 8, torch.float64), (5, 3, torch.float32)])
def test_tall_gram_bordered(dv, n, K, dt):
    """fdmd_tall_gram_bordered: [X^T X | X^T s_m] in one pass (the border rides in
    the diagonal warp tiles of the symmetric panel Gram when K % 8 == 0, inside
    the last block column otherwise; tiny / unaligned operands fall back to the
    symmetric Gram + tall_tdot) against fp64 products; bitwise repeatable; beta
    accumulation (streamed upload); identical to the separate Gram + border."""
    rng = np.random.default_rng(n + K)
    S = rng.standard_normal((n, K + 1)).astype(np.float32 if dt == torch.float32 else np.float64)
    Sd = S.astype(np.float64)
    want = Sd[:, :K].T @ Sd
    St = _tall_from(dv, S, "row", dt)
    ops = dv.get_ops()
    G = ops.tall_gram_bordered(St, K)
    assert G.shape == (K, K + 1)
    tol = 1e-12 * np.abs(Sd).max() ** 2 * n
    np.testing.assert_allclose(G.cpu().numpy(), want, rtol=1e-12, atol=tol)
    np.testing.assert_allclose(G[:, :K].cpu().numpy(), G[:, :K].t().cpu().numpy(), rtol=1e-14, atol=tol * 1e-2)
    assert torch.equal(G, ops.tall_gram_bordered(St, K))
    acc = G.clone()
    ops.tall_gram_bordered(St, K, out=acc, beta=1.0)
    np.testing.assert_allclose(acc.cpu().numpy(), 2 * want, rtol=1e-12, atol=2 * tol)
    G2 = ops.tall_gram(St, St, K1=K, K2=K, symmetric=True)
    np.testing.assert_allclose(G[:, :K].cpu().numpy(), G2.cpu().numpy(), rtol=1e-13, atol=tol * 0.1)
    y = ops.tall_tdot(St, K, K)
    np.testing.assert_allclose(G[:, K].cpu().numpy(), y.cpu().numpy(), rtol=1e-12, atol=tol)


@pytest.mark.parametrize("n,r,units", [(300007, 200, 100), (70001, 150, 75), (256 * 148 * 3, 64, 100), (5000, 200, 40)])
def test_tc_decode_fused_pair_stats(dv, n, r, units):
    """The modes product's frame epilogue also takes max_i |phi_u[i]|^2 and the
    first row attaining it (fdmd_tc_decode_pairstats): bitwise equal to
    pair_stats over the written table, frames identical to plain tc_decode;
    batches of <= 128 columns report `not fused` (None)."""
    rng = np.random.default_rng(n + units)
    ops = dv.get_ops()
    Ut = _tall_from(dv, rng.standard_normal((n, r)).astype(np.float32) / np.sqrt(n), "col", torch.float32)
    tcb = ops.tc_basis(Ut)
    coef = torch.as_tensor(rng.standard_normal((r, 2 * units)), device="cuda")
    raw = dv.alloc_tall(n, 2 * units, torch.float32, "col")
    ref = dv.alloc_tall(n, 2 * units, torch.float32, "col")
    ops.tc_decode(tcb, coef, out=ref.buf[: 2 * units])
    st = ops.tc_decode_pairstats(tcb, coef, raw.buf[: 2 * units], units, row_offset=17)
    if 2 * units <= 128:
        assert st is None
        assert torch.equal(raw.buf[: 2 * units, :n], ref.buf[: 2 * units, :n])
        return
    assert st is not None and torch.equal(raw.buf[: 2 * units, :n], ref.buf[: 2 * units, :n])
    want = ops.pair_stats(ref, units, row_offset=17)
    # the fused magnitudes are evaluated in f32: the maximum agrees to f32 rounding and
    # the argmax is a row whose f64 magnitude is within that rounding of the maximum
    np.testing.assert_allclose(st[:, 1].cpu().numpy(), want[:, 1].cpu().numpy(), rtol=3e-7)
    rows = (st[:, 2] - 17).long()
    ar = torch.arange(units, device="cuda")
    mag = ref.buf[2 * ar, rows].double() ** 2 + ref.buf[2 * ar + 1, rows].double() ** 2
    assert torch.all(mag >= want[:, 1] * (1 - 3e-7))
    assert float((st[:, 2] == want[:, 2]).double().mean()) >= 0.98
    np.testing.assert_allclose(st[:, 0].cpu().numpy(), want[:, 0].cpu().numpy(), rtol=3e-7)
    # planted ties: the first row wins
    raw.buf[: 2 * units].zero_()
    Z = torch.zeros((n, r), dtype=torch.float32)
    Z[5, 0] = Z[n - 3, 0] = 1.0
    tz = ops.tc_basis(_tall_from(dv, Z.numpy(), "col", torch.float32))
    c2 = torch.zeros((r, 2 * units), dtype=torch.float64, device="cuda")
    c2[0, :] = 1.0
    st2 = ops.tc_decode_pairstats(tz, c2, raw.buf[: 2 * units], units)
    assert torch.all(st2[:, 2] == 5.0) and torch.all(st2[:, 1] == 2.0) and torch.all(st2[:, 0] == 4.0)


@pytest.mark.parametrize("l,T,cond", [(200, 200, 1.2e4), (160, 201, 1e6), (20, 100, 10.0), (1, 5, 1.0)])
def test_svd_small_gesvdp(dv, l, T, cond):
    """fdmd_svd_small (cuSOLVER gesvdp, stream-ordered): the thin SVD of the fit's
    small projected matrix B (a strided column window of Q^T S) against LAPACK."""
    rng = np.random.default_rng(l + T)
    U0, _ = np.linalg.qr(rng.standard_normal((l, l)))
    V0, _ = np.linalg.qr(rng.standard_normal((T, l)))
    sv = cond ** (-np.arange(l) / max(l - 1, 1))
    full = np.zeros((l, T + 3))
    full[:, :T] = (U0 * sv) @ V0.T
    Bt = torch.as_tensor(full, device="cuda")[:, :T]          # non-contiguous window, like QtS[:, :T]
    Ub, s, Vh, info = dv.get_ops().svd_small(Bt)
    assert int(info.item()) == 0
    s_h = s.cpu().numpy()
    np.testing.assert_allclose(s_h, sv, rtol=1e-10 * cond, atol=0)
    assert np.all(np.diff(s_h) <= 0)
    rec = (Ub * s[None, :]) @ Vh
    assert float((rec - Bt).abs().max()) <= 1e-13
    eye = torch.eye(l, dtype=torch.float64, device="cuda")
    assert float((Ub.t() @ Ub - eye).abs().max()) <= 1e-12 and float((Vh @ Vh.t() - eye).abs().max()) <= 1e-12
    assert torch.equal(Bt, torch.as_tensor(full, device="cuda")[:, :T])   # input untouched


@pytest.mark.parametrize("nv", [1, 3, 8])
def test_colmajor_dot(dv, nv):
    rng = np.random.default_rng(nv)
    n, r = 123457, 40
    D = rng.standard_normal((n, r))
    U = rng.standard_normal((nv, n))
    Dt = _tall_from(dv, D, "col", torch.float64)
    y = dv.get_ops().colmajor_dot(Dt, torch.as_tensor(U, device="cuda")).cpu().numpy()
    np.testing.assert_allclose(y, D.T @ U.T, rtol=1e-11, atol=1e-11 * np.abs(D.T @ U.T).max())


def test_table_apply_and_residual(dv):
    rng = np.random.default_rng(9)
    n, U, m = 20000, 5, 12
    R = rng.standard_normal((n, 2 * U))
    Rt = _tall_from(dv, R, "col", torch.float64)
    src = [0, 0, 3, 4, 2]
    al = rng.standard_normal(5)
    be = rng.standard_normal(5)
    Dt = dv.alloc_tall(n, 5, torch.float64, "col")
    dv.get_ops().table_apply(Rt, src, al, be, Dt, 5)
    D = Dt.view().cpu().numpy()
    want = np.stack([al[j] * R[:, 2 * src[j]] + be[j] * R[:, 2 * src[j] + 1] for j in range(5)], axis=1)
    np.testing.assert_allclose(D, want, rtol=1e-14, atol=1e-14)
    for dt in (torch.float64, torch.float32):
        Ri = _tall_from(dv, R, "col", dt)
        Ti = dv.get_ops().table_apply_inplace(Ri, src, al, be, 5)
        assert Ti.k == 5 and Ti.buf.data_ptr() == Ri.buf.data_ptr()
        Rd = R.astype(np.float32).astype(np.float64) if dt == torch.float32 else R
        want_i = np.stack([al[j] * Rd[:, 2 * src[j]] + be[j] * Rd[:, 2 * src[j] + 1] for j in range(5)], axis=1)
        tol = 1e-6 if dt == torch.float32 else 1e-14
        np.testing.assert_allclose(Ti.view().double().cpu().numpy(), want_i, rtol=tol, atol=tol)
    S = rng.standard_normal((n, m))
    St = _tall_from(dv, S, "row", torch.float64)
    F = rng.standard_normal((5, m - 1))
    out = dv.get_ops().residual(St, Dt, torch.as_tensor(F, device="cuda"), 5, m - 1).cpu().numpy()
    np.testing.assert_allclose(out[0], np.sum((S[:, 1:] - D @ F) ** 2), rtol=1e-12)
    np.testing.assert_allclose(out[1], np.sum(S[:, 1:] ** 2), rtol=1e-12)


@pytest.mark.parametrize("n", [6, 50, 200])
def test_geev(dv, n):
    rng = np.random.default_rng(n)
    K = rng.standard_normal((n, n))
    w, V = dv.get_ops().geev(torch.as_tensor(K, device="cuda"))
    assert np.linalg.norm(K @ V - V * w) <= 1e-10 * np.linalg.norm(K) * np.linalg.norm(V)
    ref = np.linalg.eigvals(K)
    from conftest import match_eigs
    assert match_eigs(w, ref) <= 1e-10 * np.abs(ref).max()


def test_synth3d_matches_host(dv):
    from paper_2502_05339_b200 import synth
    p = synth.config_params(1, seed=5, grid=12)
    p.dtype = np.float64
    Xh = synth.generate_host(p).astype(np.float64)
    sx, sy, sz, A = [torch.as_tensor(np.ascontiguousarray(t), device="cuda") for t in p.sep_tables()]
    out = dv.alloc_tall(p.n, p.m, torch.float64, "row")
    dv.get_ops().synth3d((sx, sy, sz, A), p.m, p.noise, synth.noise_key(p.seed), 0, p.n, out)
    Xd = out.view().cpu().numpy()
    assert np.abs(Xd - Xh).max() <= 1e-11 * np.abs(Xh).max()
