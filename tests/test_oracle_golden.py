"""Pin the CPU oracle (oracle/sigkern_oracle.py) against the reference's own outputs.

The golden vectors were produced by running the reference itself
(tests/golden/make_golden.py). CPU only.
"""

import numpy as np
import pytest

from conftest import oracle_static
from oracle import sigkern_oracle as O


def test_gen_brownian_bitwise(brownian_golden):
    for key in ("n3_L10_d5_s1", "n2_L256_d16_s1", "n2_L256_d16_s2", "n1_L2_d1_s7"):
        n, L, d, s = [int(t[1:]) for t in key.split("_")]
        assert np.array_equal(O.gen_brownian(n, L, d, s), brownian_golden[key]), key
    assert np.array_equal(O.gen_brownian(2, 12, 2, 31, ("a", "b")), brownian_golden["child_path"])


def test_gen_brownian_window_stable():
    full = O.gen_brownian(6, 9, 3, 4)
    assert np.array_equal(O.gen_brownian(3, 9, 3, 4, start=2), full[2:5])


def test_gram_cases_match_reference(gram_cases):
    worst = 0.0
    for name, X, Y, c, K_ref in gram_cases:
        if name.startswith("bench_c5") or name.startswith("bench_c4"):
            continue  # large; covered by test_bench_blocks_match_reference
        K = O.gram(X, Y, sp=oracle_static(c), M=c["n_levels"], p=c["order"],
                   difference=c["difference"], normalization=c["normalization"])
        assert K.shape == K_ref.shape
        rel = np.abs(K - K_ref) / np.maximum(np.abs(K_ref), 1e-300)
        worst = max(worst, float(rel.max()))
        assert np.allclose(K, K_ref, rtol=1e-12, atol=1e-14), name
    assert worst < 1e-12


@pytest.mark.parametrize("name", ["bench_c4", "bench_c5"])
def test_bench_blocks_match_reference(gram_cases, name):
    _, X, Y, c, K_ref = gram_cases.get(name)
    K = O.gram(X, Y, sp=oracle_static(c), M=c["n_levels"], p=c["order"],
               normalization=c["normalization"])
    assert np.array_equal(K, K_ref)


def test_levels_dp_bitwise(levels_golden):
    z = levels_golden
    for t in range(24):
        A = z[f"dp{t}__A"]
        M, p = (int(v) for v in z[f"dp{t}__Mp"])
        assert np.array_equal(O.levels_dp(A, M, p), z[f"dp{t}__dp"]), t
        assert np.allclose(O.levels_bruteforce(A, M, p), z[f"dp{t}__bf"], rtol=1e-12, atol=1e-14)
    mats = list(z["perlevel__A"])
    assert np.array_equal(O.levels_dp(mats, 3, 2), z["perlevel__dp"])
    assert np.array_equal(O.levels_dp(z["batched__A"], 4, 2), z["batched__dp"])


def test_increments_bitwise(levels_golden):
    z = levels_golden
    for kind in O.KINDS:
        sp = O.static_params(kind, bandwidth=1.2)
        x, y = z[f"inc_{kind}__x"], z[f"inc_{kind}__y"]
        assert np.array_equal(O.increments(sp, x, y), z[f"inc_{kind}__A"]), kind
        assert np.array_equal(O.increments(sp, x, y, difference=False), z[f"inc_{kind}__G"]), kind


def test_hand_values():
    # test_acceptance.py:90-100: k1 = 6; k2 = 0 at p=1, 9 at p=2
    lin = O.static_params("linear")
    x = np.array([[0.0], [1.0], [3.0]])
    y = np.array([[0.0], [2.0]])
    A = O.increments(lin, x, y)
    assert O.levels_dp(A, 2, 1)[1] == pytest.approx(6.0)
    assert O.levels_dp(A, 2, 1)[2] == 0.0
    assert O.levels_dp(A, 2, 2)[2] == pytest.approx(9.0)
    assert O.levels_bruteforce(A, 2, 2)[2] == pytest.approx(9.0)


def test_oracle_median_heuristic_golden():
    """The oracle's median_heuristic restatement reproduces the reference's values."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "median.npz"))
    for name in sorted({k.split("__")[0] for k in z.files}):
        got = O.median_heuristic(z[f"{name}__X"], max_pairs=int(z[f"{name}__max_pairs"]))
        assert got == float(z[f"{name}__median"]), name  # same numpy ops: bitwise


def _pde_cases():
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "pde.npz"))
    for name in sorted({k.split("__")[0] for k in z.files}):
        kind = str(z[f"{name}__kind"])
        par = float(z[f"{name}__param"])
        sp = O.static_params(kind, **({"scale": par} if kind == "linear" else {"bandwidth": par}))
        Y = z[f"{name}__Y"] if f"{name}__Y" in z.files else None
        yield name, z[f"{name}__X"], Y, sp, bool(z[f"{name}__diff"]), str(z[f"{name}__norm"]), \
            z[f"{name}__K"], kind, par


def test_oracle_pde_golden():
    """The oracle's row-streamed PDE restatement reproduces the reference (kernels.py:334-507)."""
    for name, X, Y, sp, diff, norm, K, _, _ in _pde_cases():
        got = O.pde_gram(X, Y, sp=sp, difference=diff, normalization=norm)
        assert np.allclose(got, K, rtol=1e-12, atol=0), name


def test_rfsf_exact_gram_oracle_matches_reference(rfsf_cases):
    assert len(rfsf_cases) >= 10
    for c in rfsf_cases:
        K = O.rfsf_exact_gram(c.oracle_slots(), c.X, c.Y, M=c.M, p=c.p,
                              difference=c.difference, normalize=c.normalize)
        assert K.shape == c.K.shape, c.name
        assert np.allclose(K, c.K, rtol=1e-11, atol=1e-13), c.name


def test_rfsf_criterion06_lifted_equals_direct(rfsf_cases):
    # test_acceptance.py:183-208: the lifted dual Gram equals the materialised
    # rfsf_full feature inner products (max abs 1e-8)
    n = 0
    for c in rfsf_cases:
        if c.direct is None:
            continue
        n += 1
        assert np.abs(c.direct - c.K).max() <= 1e-8, c.name
    assert n >= 8


def test_rfsf_fit_rff_reproduces_reference(rfsf_cases):
    # fit_sig_features' rff slots are host-side numpy sampling: bitwise the reference's
    from paper_2501_07145_b200 import SeedStream
    from paper_2501_07145_b200.features import fit_sig_features
    for c in rfsf_cases:
        if c.kind != "rff":
            continue
        st = fit_sig_features(c.state().config, c.X, SeedStream(23, (c.name,)))
        assert len(st.slot_states) == c.M
        for a, s in enumerate(st.slot_states):
            assert np.array_equal(s.weights, c.slots[a]["weights"]), (c.name, a)
            assert s.out_dim == 2 * c.D


def test_c3_far_block_matches_reference():
    """The far-end c3 golden block (rows/cols 8168-8191 of the full inputs): the
    window of the prefix-stable generator reproduces the reference's slice, and the
    oracle reproduces its 24 x 24 Gram (levelwise and unnormalised)."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "c3_far.npz"))
    X = O.gen_brownian(24, 256, 16, 1, start=8168)
    Y = O.gen_brownian(24, 256, 16, 2, start=8168)
    assert np.array_equal(X, z["X"]) and np.array_equal(Y, z["Y"])
    for norm in ("levelwise", "none"):
        K = O.gram(X[:6], Y[:5], M=5, p=1, normalization=norm, n_threads=O.host_threads())
        assert np.allclose(K, z[f"K_{norm}"][:6, :5], rtol=1e-12, atol=0), norm
