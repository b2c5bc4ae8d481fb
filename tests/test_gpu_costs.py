"""GPU parity of the SA cost functions (static Hagan/Obloj Eq. 7, Osajima
Eq. 8) against the compiled reference: identical parameter vectors, values
within 1e-12 relative in FP64 (mixed: |d| <= 1e-12 * max(|c|, 1e-8), since a
perfect fit has cost -> 0 where relative error is meaningless).

Where the reference's own Case I closed forms cancel (x = decay*T just above
the 0.25 series switch, analytics.cpp:47-67: up to 6e3x for f_eta2) a one-ulp
difference between glibc's and libdevice's exp moves the reference value by
more than 1e-12; there the bound is twice the reference's own one-ulp
sensitivity, measured by the oracle (orc_cost_sensitivity).  The fraction of
vectors needing that allowance is asserted to stay below 0.1%."""
import numpy as np
import pytest

import paper_2407_20713_b200 as pkg

pytestmark = pytest.mark.gpu

TOL = 1e-12


def mixed_err(got, want):
    return np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-8))


def static_vectors(n, seed):
    rng = np.random.default_rng(seed)
    # default box, calibration.cpp:24-31
    return np.column_stack([rng.uniform(1e-4, 2, n), rng.uniform(0, 1, n), rng.uniform(1e-4, 10, n),
                            rng.uniform(-1, 1, n)])


def case1_vectors(n, seed):
    rng = np.random.default_rng(seed)
    P = np.column_stack([rng.uniform(1e-4, 2, n), rng.uniform(0, 1, n), rng.uniform(-1, 1, n),
                         rng.uniform(1e-4, 10, n), rng.uniform(0, 150, n), rng.uniform(0, 150, n)])
    # a quarter in the Taylor-series branch (x = decay*T < 0.25), analytics.cpp:47-67
    k = n // 4
    P[:k, 4:] = rng.uniform(0, 0.1, (k, 2))
    P[k:2 * k, 1] = 1.0  # beta = 1 (pow(f, 0) = 1 exactly)
    return P


@pytest.mark.parametrize("fixture", ["eq_surface", "fx_surface"])
def test_static_cost_parity(engine, ref, request, fixture):
    surface = request.getfixturevalue(fixture)
    P = static_vectors(10_000, 42)
    for sl in range(len(surface.slices)):
        got = engine.cost_batch(pkg.MODEL_STATIC, surface, P, slice=sl)
        want = ref.cost_static(surface, sl, P)
        err = mixed_err(got, want)
        assert err < TOL, f"slice {sl}: {err:.3e}"


def test_static_cost_parity_small_and_large_slices(engine, ref):
    """The factored slice cost (slice_qr.hpp) on slices of 1, 2, 3 quotes
    (rank-deficient factors: R has zero rows), 4 (square), and 600 quotes."""
    rng = np.random.default_rng(7)
    slices = []
    for n in (1, 2, 3, 4, 600):
        K = np.sort(rng.uniform(0.6, 1.5, n))
        v = rng.uniform(0.08, 0.6, n)
        slices.append(pkg.VolSlice(0.25 + 0.5 * len(slices), 0.01, 0.002,
                                   [pkg.VolQuote(float(k), float(x)) for k, x in zip(K, v)]))
    surface = pkg.VolSurface(1.0, slices)
    P = static_vectors(4_000, 44)
    for sl in range(len(slices)):
        got = engine.cost_batch(pkg.MODEL_STATIC, surface, P, slice=sl)
        want = ref.cost_static(surface, sl, P)
        err = mixed_err(got, want)
        assert err < TOL, f"slice {sl}: {err:.3e}"


@pytest.mark.parametrize("fixture", ["eq_surface", "fx_surface"])
def test_case1_cost_parity(engine, ref, orc, request, fixture):
    from oracles import cost_sensitivity

    surface = request.getfixturevalue(fixture)
    P = case1_vectors(10_000, 43)
    got = engine.cost_batch(pkg.MODEL_CASE1, surface, P, slice=-1)
    want = ref.cost_case1(surface, P)
    d = np.abs(got - want)
    plain = d / np.maximum(np.abs(want), 1e-8)
    sens = cost_sensitivity(orc, pkg.MODEL_CASE1, surface, -1, P)
    bound = np.maximum(TOL * np.maximum(np.abs(want), 1e-8), 2.0 * sens)
    print(f"case1 {fixture}: max rel {plain.max():.2e}, frac > 1e-12 {np.mean(plain > TOL):.4%}, "
          f"max d/bound {np.max(d / bound):.2f}")
    assert np.all(d <= bound)
    assert np.mean(plain > TOL) < 1e-3


def test_static_vols_match_reference_formula(engine, ref, eq_surface):
    P = static_vectors(64, 5)
    for sl in range(4):
        got = engine.implied_vol_batch(pkg.MODEL_STATIC, eq_surface, P, slice=sl)
        f = eq_surface.forward(sl)
        T = eq_surface.slices[sl].maturity
        for i in range(0, 64, 7):
            for j, q in enumerate(eq_surface.slices[sl].quotes):
                want = ref.static_vol(P[i], q.strike, f, T)
                assert abs(got[i, j] - want) <= 1e-13 * abs(want)


def test_nu_zero_gives_alpha(engine):
    # proj/tests/test_analytics.cpp:28-36: nu = 0, beta = 1 => sigma = alpha (1e-14)
    s = pkg.VolSurface(100.0, [pkg.VolSlice(1.0, 0.0, 0.0, [pkg.VolQuote(k, 0.2) for k in (80.0, 100.0, 125.0)])])
    v = engine.implied_vol_batch(pkg.MODEL_STATIC, s, np.array([[0.25, 1.0, 0.0, 0.3]]), slice=0)
    assert np.max(np.abs(v - 0.25)) < 1e-14


def test_case1_constant_params_equal_static(engine, eq_surface):
    # acceptance c1 (proj/tests/acceptance.cpp:88-110): a = b = 0 reduces Eq. 8 to Eq. 7
    rng = np.random.default_rng(101)
    for _ in range(10):
        a, b, nu, rho = 0.05 + 0.6 * rng.random(), rng.random(), 0.05 + rng.random(), -0.99 + 1.9 * rng.random()
        st = engine.implied_vol_batch(pkg.MODEL_STATIC, eq_surface, np.array([[a, b, nu, rho]]), slice=2)
        dy = engine.implied_vol_batch(pkg.MODEL_CASE1, eq_surface, np.array([[a, b, rho, nu, 0.0, 0.0]]))
        q0 = sum(len(s.quotes) for s in eq_surface.slices[:2])
        d = dy[0, q0:q0 + st.shape[1]]
        assert np.max(np.abs(d - st[0]) / st[0]) < 1e-12


def test_published_case1_vols(engine, eq_surface, fx_surface):
    # acceptance c4/c5: Table 6 / Table 9 model vols to 1e-3 vol points
    cases = [
        (eq_surface, [0.294722, 1.0, -1.0, 0.388539, 0.001, 0.131466], [4, 10, 16],
         [[31.7628, 29.2166, 27.1094], [31.3150, 28.8068, 26.7345], [30.7756, 28.3187, 26.2941],
          [29.6026, 27.2549, 25.3308]]),
        (fx_surface, [0.155464, 0.971908, -0.642617, 0.800275, 0.001, 2.6093], [3, 9, 15],
         [[17.0683, 15.4197, 14.3171], [17.4751, 15.3398, 14.0914], [17.6324, 15.2020, 14.0396],
          [17.3887, 15.1075, 14.2853]]),
    ]
    for surface, p, cols, want in cases:
        v = engine.implied_vol_batch(pkg.MODEL_CASE1, surface, np.array([p]))[0]
        off = 0
        for i, s in enumerate(surface.slices):
            for j, c in enumerate(cols):
                assert abs(100 * v[off + c] - want[i][j]) < 1e-3
            off += len(s.quotes)


def test_domain_errors(engine, eq_surface):
    with pytest.raises(pkg.DomainError):
        engine.cost_batch(pkg.MODEL_STATIC, eq_surface, np.array([[0.0, 1.0, 0.5, 0.0]]), slice=0)
    with pytest.raises(pkg.DomainError):
        engine.cost_batch(pkg.MODEL_CASE1, eq_surface, np.array([[0.3, 1.0, -0.5, 0.0, 0.1, 0.1]]))
    with pytest.raises(pkg.OutOfRangeError):
        engine.cost_batch(pkg.MODEL_STATIC, eq_surface, np.array([[0.3, 1.0, 0.5, 0.0]]), slice=9)


def feasible_case2_vectors(ref, n, seed, horizon):
    rng = np.random.default_rng(seed)
    lo = np.array([1e-4, 0, -1, -15, -1, 1e-4, -15, -1, 0, 0])
    hi = np.array([2, 1, 1, 15, 1, 10, 15, 1, 150, 150])
    out = []
    while len(out) < n:
        P = lo + (hi - lo) * rng.random((4 * n, 10))
        P[:, 3] *= rng.random(4 * n) ** 3  # favour the feasible region
        P[:, 6] *= rng.random(4 * n) ** 3
        P = np.column_stack([P, np.full(len(P), horizon)])
        out.extend(P[ref.case2_feasible(P)])
    return np.array(out[:n])


@pytest.mark.parametrize("fixture", ["eq_surface", "fx_surface"])
def test_case2_formula_cost_parity(engine, ref, request, fixture):
    """calibrate_case2_formula objective (calibration.cpp:497-520): nested GL
    eta2^2 + Black-Scholes, CTA-cooperative on the GPU vs the reference."""
    from oracles import ref_cost_case2_formula

    surface = request.getfixturevalue(fixture)
    H = surface.slices[-1].maturity
    P = feasible_case2_vectors(ref, 300, 5, H)
    pub = np.array([[0.296790, 1.0, -0.360610, 15.0, -0.715716, 0.000100, -8.969205, 0.847244, 15.0, 15.0, H],
                    [0.154037, 1.0, -0.693682, 0.345973, -0.200342, 7.541424, -0.992551, 0.339807, 0.0, 150.0, H]])
    P = np.vstack([pub[ref.case2_feasible(pub)], P])
    got = engine.cost_batch(3, surface, P)
    want = ref_cost_case2_formula(ref, surface, P)
    assert np.array_equal(got == 1e10, want == 1e10)  # same "left its validity range" verdicts
    ok = want != 1e10
    rel = np.abs(got[ok] - want[ok]) / np.maximum(np.abs(want[ok]), 1e-8)
    print(f"case2 formula {fixture}: {ok.sum()} finite, max rel {rel.max():.2e}")
    assert rel.max() < 1e-10


def test_case2_model_vols_match_reference(engine, ref):
    """Case II model vols dynamic_implied_vol(dyn_coeffs_case2(p, T, 64), ...)
    (the smile command, sabr_cli.cpp:234-243) on the 20x30 synthetic surface,
    which the reference generated from exactly these vols at the FX fit."""
    import os

    surface = pkg.parse_surface(os.path.join(os.path.dirname(__file__), "data", "synth20x30.csv"))
    H = surface.slices[-1].maturity
    fx_fit = [0.154037, 1.0, -0.693682, 0.345973, -0.200342, 7.541424, -0.992551, 0.339807, 0.0, 150.0, H]
    P = np.vstack([fx_fit, feasible_case2_vectors(ref, 40, 8, H)])
    got = engine.implied_vol_batch(pkg.MODEL_CASE2, surface, P)
    worst = 0.0
    for i, p in enumerate(P):
        off = 0
        for s, sl in enumerate(surface.slices):
            c = ref.dyn_coeffs_case2(p, sl.maturity, 64)
            f = surface.forward(s)
            for j, q in enumerate(sl.quotes):
                want = ref.dynamic_vol(c, p[0], p[1], q.strike, f, sl.maturity)
                if np.isfinite(want) and want > 0:
                    worst = max(worst, abs(got[i, off + j] - want) / abs(want))
            off += len(sl.quotes)
    # eta2^2 is a nested 64x64-node quadrature summed in another order (CTA
    # reduction): measured worst 1.4e-12 relative over 41 vectors x 600 quotes
    assert worst < 1e-11, worst
    # the fixture's own vols (written as 100*vol in shortest form) at the fit
    market = np.array([q.vol for sl in surface.slices for q in sl.quotes])
    assert np.max(np.abs(got[0] - market) / market) < 1e-14
