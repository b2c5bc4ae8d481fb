"""Pins the oracle restatement (oracle/sabr_oracle.c) against the golden
vectors the unmodified reference produced (tests/golden/golden.json, made by
tests/golden/make_golden.py from oracle/_ref) and, where oracle/_ref is built,
against the reference live.  Integer/stream results must be bit-identical; all
floating point results are compared bit-for-bit too (same libm, same
operation order, no FMA contraction)."""
import json
import os

import numpy as np
import pytest

import paper_2407_20713_b200 as pkg
from paper_2407_20713_b200 import _abi as A
from oracles import DATA_DIR, Ref, Restate, atm_vol_guess, have_ref, have_restate

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))

pytestmark = pytest.mark.skipif(not have_restate(), reason="oracle restatement not built")


def fx(v):
    if isinstance(v, list):
        return np.array([fx(x) for x in v])
    return float.fromhex(v)


def golden_surface(name):
    g = GOLDEN["surfaces"][name]
    slices = [pkg.VolSlice(fx(T), fx(r), fx(y), [pkg.VolQuote(fx(k), fx(v)) for k, v in qs])
              for T, r, y, qs in g["slices"]]
    return pkg.VolSurface(fx(g["spot"]), slices)


@pytest.fixture(scope="module")
def orc():
    return Restate()


@pytest.mark.parametrize("name", ["eurostoxx50", "eurusd"])
def test_surface_loader_matches_reference_parser(name):
    # the engine's C++ loader (sabr_surface_csv_*) vs io::parse_surface's golden output
    s = pkg.parse_surface(os.path.join(DATA_DIR, name + ".csv"))
    g = golden_surface(name)
    assert s.spot == g.spot and len(s.slices) == len(g.slices)
    for a, b in zip(s.slices, g.slices):
        assert (a.maturity, a.rate, a.dividend) == (b.maturity, b.rate, b.dividend)
        assert [(q.strike, q.vol) for q in a.quotes] == [(q.strike, q.vol) for q in b.quotes]


@pytest.mark.parametrize("name", ["eurostoxx50", "eurusd"])
def test_static_cost_golden(orc, name):
    s = golden_surface(name)
    P = fx(GOLDEN["cost_static"]["params"])
    for sl in range(4):
        want = fx(GOLDEN["cost_static"][name][sl])
        assert np.array_equal(orc.cost_static(s, sl, P), want)


@pytest.mark.parametrize("name", ["eurostoxx50", "eurusd"])
def test_case1_cost_golden(orc, name):
    s = golden_surface(name)
    P = fx(GOLDEN["cost_case1"]["params"])
    assert np.array_equal(orc.cost_case1(s, P), fx(GOLDEN["cost_case1"][name]))


def test_case2_feasibility_golden(orc):
    P = fx(GOLDEN["case2_feasible"]["params"])
    want = np.array(GOLDEN["case2_feasible"]["feasible"])
    assert np.array_equal(orc.case2_feasible(P), want)
    assert 0 < want.sum() < len(want)  # both outcomes are exercised


def test_xoshiro_streams_golden(orc):
    import ctypes as C

    class X(C.Structure):
        _fields_ = [("s", C.c_uint64 * 4)]

    orc.lib.orc_xoshiro_uniform.restype = C.c_double
    for key, vals in GOLDEN["xoshiro"].items():
        seed, stream = (int(v) for v in key.split("_"))
        g = X()
        orc.lib.orc_xoshiro_init(C.byref(g), C.c_uint64(seed), C.c_uint64(stream))
        got = [orc.lib.orc_xoshiro_uniform(C.byref(g)) for _ in range(8)]
        assert got == list(fx(vals))


def test_philox_known_answers(orc):
    """Random123 Philox4x32-10 known-answer vectors (kat_vectors)."""
    import ctypes as C

    cases = [((0, 0, 0, 0), 0, (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
             ((0xFFFFFFFF,) * 4, 0xFFFFFFFFFFFFFFFF, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
             ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), 0x299F31D0A4093822,
              (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in cases:
        c = (C.c_uint32 * 4)(*ctr)
        out = (C.c_uint32 * 4)()
        orc.lib.orc_philox4x32(c, C.c_uint64(key), out)
        assert tuple(out) == want


@pytest.mark.parametrize("name", list(GOLDEN["anneal_builtin"]))
def test_annealer_builtin_golden(orc, name):
    g = GOLDEN["anneal_builtin"][name]
    s = pkg.AnnealingSchedule(**g["schedule"])
    r = orc.minimize_builtin(g["objective"], g["lower"], g["upper"], s, g["start"], predicate=g["predicate"])
    assert r.evals == g["evals"]
    assert r.best_value == fx(g["best_value"])
    assert r.best_point == list(fx(g["best_point"]))
    assert [(t, f) for t, f in r.temperature_trace] == [(fx(t), fx(f)) for t, f in g["trace"]]


@pytest.mark.parametrize("seed", ["1", "2", "3"])
def test_static_T1_trajectory_golden(orc, seed):
    """C1 schedule: 412 levels x 32 chains, 1,000,001 evals — the whole
    trajectory reproduces bit for bit."""
    g = GOLDEN["anneal_static_c1"][seed]
    eq = golden_surface("eurostoxx50")
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=int(seed))
    r = orc.minimize_cost(A.MODEL_STATIC, eq, 0, [1e-4, 0, 1e-4, -1], [2, 1, 10, 1], s, list(fx(g["start"])))
    assert list(fx(g["start"])) == [atm_vol_guess(eq, 0), 1.0, 0.5, -0.3]
    assert r.evals == g["evals"] == 1_000_001
    assert r.best_value == fx(g["best_value"]) and r.best_point == list(fx(g["best_point"]))
    assert [f for _, f in r.temperature_trace] == list(fx(g["trace_f"]))


@pytest.mark.parametrize("name", ["static", "case1", "case2"])
def test_mc_streams_golden(orc, name):
    g = GOLDEN["mc"][name]
    cls = {"static": pkg.StaticSabrParams, "case1": pkg.CaseIParams, "case2": pkg.CaseIIParams}[name]
    p = cls(*g["params"])
    plan = pkg.SimulationPlan(num_paths=g["plan"]["num_paths"], seed=g["plan"]["seed"],
                              block_size=g["plan"]["block_size"])
    t = orc.simulate_terminals(p, 2257.37, p.alpha, 0.495890, plan)
    assert np.array_equal(t[:64], fx(g["terminals_head"]))
    assert np.array_equal(t[-64:], fx(g["terminals_tail"]))
    assert float(np.sum(t)) == fx(g["terminals_sum"])
    est = orc.price_european_batch(p, 2257.37, [2000.0, 2257.37, 2500.0], 0.018196, 0.034516, 0.495890, plan)
    for e, (v, se) in zip(est, g["prices"]):
        assert e.value == fx(v) and e.std_error == fx(se)


def test_black_scholes_matches_reference_fixture(orc):
    # test_calibration.cpp:84-97: ATM 3m equity quote 29.79% -> 134.605
    eq = golden_surface("eurostoxx50")
    sl = eq.slices[0]
    p = orc.black_scholes_call(eq.spot, sl.quotes[10].strike, sl.rate, sl.dividend, sl.maturity, sl.quotes[10].vol)
    assert abs(p - 134.605) <= 2e-5 * 134.605


def bs_contracts(n, seed=9):
    """test_black_scholes.cpp:10-23 style random contracts (spot, K, r, y, T, vol)."""
    rng = np.random.default_rng(seed)
    spot = 50.0 + 4000.0 * rng.uniform(size=n)
    return (spot, spot * (0.7 + 0.6 * rng.uniform(size=n)), 0.05 * rng.uniform(size=n),
            0.05 * rng.uniform(size=n), 0.1 + 2.0 * rng.uniform(size=n), 0.05 + 0.5 * rng.uniform(size=n))


def test_implied_vol_round_trip(orc):
    # test_black_scholes.cpp:10-23: price -> implied vol recovers vol to 1e-8
    # (for prices the 1e-10 price tolerance resolves: not the ~1e-18 deep OTM ones)
    for c in zip(*bs_contracts(50)):
        price = orc.black_scholes_call(*c)
        if price > 1e-8 * c[0]:
            assert abs(orc.implied_vol_from_price(price, *c[:5]) - c[5]) < 1e-8
    with pytest.raises(ValueError):  # outside the no-arbitrage bounds (test_black_scholes.cpp:66-69)
        orc.implied_vol_from_price(200.0, 100, 100, 0, 0, 1)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
class TestAgainstLiveReference:
    def test_black_scholes_and_implied_vol(self, orc):
        ref = Ref()
        for c in zip(*bs_contracts(300, seed=4)):
            p = orc.black_scholes_call(*c)
            assert p == ref.black_scholes_call(*c)
            assert orc.implied_vol_from_price(p, *c[:5]) == ref.implied_vol_from_price(p, *c[:5])

    def test_costs(self, orc):
        ref = Ref()
        eq = golden_surface("eurostoxx50")
        rng = np.random.default_rng(9)
        P = np.column_stack([rng.uniform(1e-4, 2, 500), rng.uniform(0, 1, 500), rng.uniform(1e-4, 10, 500),
                             rng.uniform(-1, 1, 500)])
        assert np.array_equal(orc.cost_static(eq, 1, P), ref.cost_static(eq, 1, P))

    def test_case2_mc_cost(self, orc):
        ref = Ref()
        fxs = golden_surface("eurusd")
        # the published Case II fits (acceptance.cpp:31-34), horizon 2
        P = np.array([[0.296790, 1.0, -0.360610, 15.0, -0.715716, 0.000100, -8.969205, 0.847244, 15.0, 15.0, 2.0],
                      [0.154037, 1.0, -0.693682, 0.345973, -0.200342, 7.541424, -0.992551, 0.339807, 0.0, 150.0,
                       2.0]])
        plan = pkg.SimulationPlan(num_paths=512, seed=1)
        a, b = orc.cost_case2_mc(fxs, P, plan), ref.cost_case2_mc(fxs, P, plan)
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["dt250", "dt007"])
def test_cliquet_golden(orc, name):
    from oracles import orc_price_cliquet

    g = GOLDEN["cliquet"][name]
    p = pkg.CaseIParams(0.155464, 0.971908, -0.642617, 0.800275, 0.001, 2.6093)
    plan = pkg.SimulationPlan(num_paths=3000, seed=3, block_size=1000, dt=g["dt"])
    e = orc_price_cliquet(orc, p, 1.2939, 0.010832, 0.006907, -0.02, 0.02, 0.0, 0.2, [0.25, 0.5, 0.75, 1.0], plan)
    assert e.value == fx(g["value"]) and e.std_error == fx(g["std_error"])


def test_case2_formula_golden(orc):
    from oracles import orc_cost_case2_formula, orc_dyn_coeffs_case2

    g = GOLDEN["case2_formula"]
    P = fx(g["params"])
    for p, coeffs in zip(P, g["coeffs"]):
        for T, c in zip((0.25, 1.0, 2.0), coeffs):
            assert np.array_equal(orc_dyn_coeffs_case2(orc, p, T, 8), fx(c))
    for name in ("eurusd", "eurostoxx50"):
        assert np.array_equal(orc_cost_case2_formula(orc, golden_surface(name), P), fx(g[name]))
