"""rfsf_exact_gram (features.py:446-475) on the device: the lifted level Grams
of a fitted rfsf_full map against the reference's own outputs
(tests/golden/rfsf.npz, made by tests/golden/make_rfsf_golden.py) and the CPU
oracle. Float64 path: held to 1e-10 relative, and to the reference's
criterion-06 bound (1e-8 absolute) against the materialised features."""

import numpy as np
import pytest
import torch

from oracle import sigkern_oracle as O
from paper_2501_07145_b200 import SeedStream, StaticKernelSpec, gen_brownian
from paper_2501_07145_b200.features import (SigFeatureConfig, StaticFeatureSpec,
                                            StaticFeatureState, fit_sig_features,
                                            rfsf_exact_gram, transform_static_features)

pytestmark = pytest.mark.gpu


def test_rfsf_golden(rfsf_cases):
    for c in rfsf_cases:
        K = rfsf_exact_gram(c.state(), c.X, c.Y, normalize=c.normalize)
        assert isinstance(K, np.ndarray) and K.shape == c.K.shape, c.name
        assert np.allclose(K, c.K, rtol=1e-10, atol=1e-12), (c.name, np.abs(K - c.K).max())
        if c.direct is not None:  # criterion 06 (test_acceptance.py:183-208)
            assert np.abs(K - c.direct).max() <= 1e-8, c.name
        if c.sym:
            assert np.array_equal(K, K.T), c.name


def test_rfsf_nystroem_fit_matches_reference(rfsf_cases):
    # landmarks are drawn by the same Philox stream (bitwise); the whitening comes
    # from the device landmark Gram + host eigh, so compare the Gram it yields
    n = 0
    for c in rfsf_cases:
        if c.kind != "nystroem":
            continue
        n += 1
        st = fit_sig_features(c.state().config, c.X, SeedStream(23, (c.name,)))
        for a, s in enumerate(st.slot_states):
            assert np.array_equal(s.landmarks, c.slots[a]["landmarks"]), (c.name, a)
            assert s.out_dim == c.slots[a]["whiten"].shape[1]
            W, R = s.whiten, c.slots[a]["whiten"]
            assert np.allclose(W @ W.T, R @ R.T, rtol=1e-8, atol=1e-10), (c.name, a)
        K = rfsf_exact_gram(st, c.X, c.Y, normalize=c.normalize)
        assert np.allclose(K, c.K, rtol=1e-8, atol=1e-10), c.name
    assert n >= 3


@pytest.mark.parametrize("kind", ["rff", "rff1d", "nystroem"])
def test_transform_static_features_vs_oracle(kind):
    rng = np.random.default_rng(5)
    d, D = 3, 7
    X = rng.standard_normal((4, 9, d))
    base = StaticKernelSpec(kind="rbf", bandwidth=1.4)
    spec = StaticFeatureSpec(kind=kind, n_components=D, base_kernel=base)
    W = rng.standard_normal((d, D))
    b = rng.uniform(0, 2 * np.pi, D)
    Z = rng.standard_normal((D, d))
    Wh = rng.standard_normal((D, 5))
    out = {"rff": 2 * D, "rff1d": D, "nystroem": 5}[kind]
    st = StaticFeatureState(spec, d, out, W, b if kind == "rff1d" else None,
                            Z if kind == "nystroem" else None, Wh if kind == "nystroem" else None)
    U = transform_static_features(st, X)
    R = O.static_features(dict(kind=kind, n_components=D, weights=W, phases=b, landmarks=Z,
                               whiten=Wh, base=O.static_params("rbf", bandwidth=1.4)), X)
    assert U.shape == R.shape == (4, 9, out)
    assert np.allclose(U, R, rtol=1e-12, atol=1e-13)
    with pytest.raises(ValueError, match="dimension mismatch"):
        transform_static_features(st, X[..., :2])


@pytest.mark.parametrize("order,diff,norm", [(1, True, False), (2, True, True),
                                             (4, True, False), (1, False, True)])
def test_rfsf_random_vs_oracle(order, diff, norm):
    X = gen_brownian(9, 17, 3, SeedStream(41)).data
    Y = gen_brownian(7, 12, 3, SeedStream(42)).data
    cfg = SigFeatureConfig(variant="rfsf_full", static=StaticFeatureSpec(kind="rff"),
                           n_components=5, projection=5, n_levels=4, order=order,
                           difference=diff)
    st = fit_sig_features(cfg, X, SeedStream(43))
    K = rfsf_exact_gram(st, X, Y, normalize=norm)
    slots = [dict(kind="rff", n_components=5, weights=s.weights) for s in st.slot_states]
    R = O.rfsf_exact_gram(slots, X, Y, M=4, p=min(order, 4), difference=diff, normalize=norm)
    assert np.allclose(K, R, rtol=1e-10, atol=1e-12)
    # symmetric: upper triangle evaluated and mirrored bit for bit; normalised diagonal is 1
    Ks = rfsf_exact_gram(st, X, normalize=True)
    assert np.array_equal(Ks, Ks.T)
    assert np.allclose(np.diag(Ks), 1.0, atol=1e-12)


def test_rfsf_torch_io_and_errors():
    X = gen_brownian(3, 6, 2, SeedStream(1)).data
    cfg = SigFeatureConfig(variant="rfsf_full", static=StaticFeatureSpec(kind="rff"),
                           n_components=3, projection=3, n_levels=3)
    st = fit_sig_features(cfg, X, SeedStream(2))
    Kt = rfsf_exact_gram(st, torch.as_tensor(X, device="cuda"))
    assert isinstance(Kt, torch.Tensor) and Kt.is_cuda
    assert np.allclose(Kt.cpu().numpy(), rfsf_exact_gram(st, X), rtol=0, atol=0)
    bad = SigFeatureConfig(variant="dp", static=StaticFeatureSpec(kind="rff"), n_components=3,
                           projection=3, n_levels=3)
    with pytest.raises(ValueError, match="rfsf_full"):
        rfsf_exact_gram(fit_sig_features(bad, X, SeedStream(2)), X)
    with pytest.raises(ValueError, match="dimension mismatch"):
        rfsf_exact_gram(st, np.zeros((2, 5, 3)))
    with pytest.raises(ValueError, match=r"\(N, L, d\)"):
        rfsf_exact_gram(st, np.zeros((5, 2)))
    st0 = fit_sig_features(SigFeatureConfig(variant="rfsf_full", static=StaticFeatureSpec(kind="rff"),
                                            n_components=3, projection=3, n_levels=0),
                           X, SeedStream(2))
    assert np.array_equal(rfsf_exact_gram(st0, X), np.ones((3, 3)))


@pytest.mark.parametrize("sym", [False, True])
def test_lifted_gram_precomputed_and_on_the_fly_agree(sym):
    """sk_lifted_gram: slot Grams precomputed by the float64 GEMM (full workspace)
    vs inner products inside the DP (minimal workspace), and a row-block call."""
    import ctypes
    from paper_2501_07145_b200 import _native
    from paper_2501_07145_b200.features import _lift
    lib = _native.load()
    X = gen_brownian(7, 13, 2, SeedStream(61)).data
    Y = gen_brownian(5, 9, 2, SeedStream(62)).data
    cfg = SigFeatureConfig(variant="rfsf_full", static=StaticFeatureSpec(kind="rff"),
                           n_components=3, projection=3, n_levels=3, order=2)
    st = fit_sig_features(cfg, X, SeedStream(63))
    UX, offs = _lift(st, torch.as_tensor(X, device="cuda"))
    UY = UX if sym else _lift(st, torch.as_tensor(Y, device="cuda"))[0]
    nx, lx, W = UX.shape
    ny, ly = UY.shape[:2]
    oc = (ctypes.c_int64 * 4)(*[int(o) for o in offs])
    stream = torch.cuda.current_stream().cuda_stream

    def run(ws_bytes, r0, r1):
        K = torch.zeros((nx if sym else r1 - r0, ny), dtype=torch.float64, device="cuda")
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
        rc = lib.sk_lifted_gram(UX.data_ptr(), nx, lx, UY.data_ptr(), ny, ly, W, oc, 3, 2, 1, 0,
                                int(sym), r0, r1, None, None, K.data_ptr(), ny, None,
                                ws.data_ptr(), ws_bytes, stream)
        assert rc == 0, lib.sk_last_error()
        return K.cpu().numpy()

    full = lib.sk_lifted_gram_workspace_bytes(nx, lx, ny, ly, 3, 2, 1)
    small = lib.sk_lifted_workspace_bytes(nx * ny, ly, 3, 2, 1)
    assert full > small
    Kg, Kf = run(full, 0, nx), run(small, 0, nx)
    assert np.allclose(Kg, Kf, rtol=1e-12, atol=1e-14)
    if not sym:
        assert np.allclose(run(full, 2, 6), Kg[2:6], rtol=1e-12, atol=1e-14)
