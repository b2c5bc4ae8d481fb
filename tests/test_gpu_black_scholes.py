"""Batched black_scholes_call / implied_vol_from_price (kernels_bs.cu) against
the compiled reference (proj/src/black_scholes.cpp:20-69) and its unit tests
(proj/tests/test_black_scholes.cpp)."""
import numpy as np
import pytest

import paper_2407_20713_b200 as pkg
from test_oracle import bs_contracts

pytestmark = pytest.mark.gpu


def test_prices_match_reference(engine, ref):
    c = bs_contracts(4000, seed=11)
    got = engine.black_scholes_call_batch(*c)
    want = np.array([ref.black_scholes_call(*x) for x in zip(*c)])
    # same operation order, no FMA: differences are the libm ulps of exp/log/erfc
    assert np.all(np.abs(got - want) <= 1e-13 * np.maximum(np.abs(want), 1e-8 * np.asarray(c[0])))
    # vol == 0: the discounted intrinsic value exactly (test_black_scholes.cpp:41-46)
    z = engine.black_scholes_call_batch(100.0, [90.0, 100.0, 110.0], 0.02, 0.01, 1.0, 0.0)
    assert list(z) == [ref.black_scholes_call(100.0, k, 0.02, 0.01, 1.0, 0.0) for k in (90.0, 100.0, 110.0)]


def test_implied_vols_match_reference(engine, ref):
    c = bs_contracts(4000, seed=12)
    price = np.array([ref.black_scholes_call(*x) for x in zip(*c)])
    # prices the 1e-10 price tolerance resolves (deep OTM ones underflow to ~1e-18 or 0,
    # where the reference's no-arbitrage check rejects or the inversion is ill-posed)
    lower = np.array([ref.black_scholes_call(*x[:5], 0.0) for x in zip(*c)])
    upper = c[0] * np.exp(-c[3] * c[4])
    # ...and not within rounding of a no-arbitrage bound, where the verdict
    # (price <= lower) rests on the last ulp of exp (glibc vs libdevice)
    ok = (price > 1e-8 * c[0]) & (price - lower > 1e-12 * c[0]) & (upper - price > 1e-12 * c[0])
    c = tuple(np.asarray(a)[ok] for a in c)
    price = price[ok]
    got = engine.implied_vol_from_price_batch(price, *c[:5])
    want = np.array([ref.implied_vol_from_price(p, *x[:5]) for p, x in zip(price, zip(*c))])
    # both stop at |BS(vol) - price| < 1e-10: a vol is determined to ~1e-10 / vega
    S, K, r, y, T, vol = c
    d1 = (np.log(S / K) + (r - y + 0.5 * vol * vol) * T) / (vol * np.sqrt(T))
    vega = S * np.exp(-y * T) * np.exp(-0.5 * d1 * d1) / np.sqrt(2 * np.pi) * np.sqrt(T)
    tol = 1e-9 + 2e-10 / vega
    assert np.all(np.abs(got - want) <= tol)   # the reference's iteration, libm ulps apart
    good = vega > 1e-1                          # the reference's own round-trip bar (1e-8)
    assert good.sum() > 3000 and np.max(np.abs(got - vol)[good]) < 1e-8
    # the published EUR/USD ATM point (test_black_scholes.cpp:26-33)
    p = ref.black_scholes_call(1.2939, 1.2950, 0.013696, 0.005894, 0.2528, 0.1470)
    iv = engine.implied_vol_from_price_batch([p], 1.2939, 1.2950, 0.013696, 0.005894, 0.2528)[0]
    assert abs(iv - 0.1470) < 1e-8


def test_errors_are_reference_domain_errors(engine):
    with pytest.raises(pkg.DomainError, match="spot, strike, maturity must be positive"):
        engine.black_scholes_call_batch([100.0, -1.0], 100.0, 0.0, 0.0, 1.0, 0.2)
    with pytest.raises(pkg.DomainError, match="vol must be nonnegative"):
        engine.black_scholes_call_batch(100.0, 100.0, 0.0, 0.0, 1.0, [0.2, -0.2])
    with pytest.raises(pkg.DomainError, match="price outside no-arbitrage bounds"):
        engine.implied_vol_from_price_batch([10.0, 200.0], 100.0, 100.0, 0.0, 0.0, 1.0)
    with pytest.raises(pkg.DomainError, match="price outside no-arbitrage bounds"):
        engine.implied_vol_from_price_batch(0.0, 100.0, 50.0, 0.02, 0.0, 1.0)
