"""Pins for the fp64 oracle (oracle/esi_oracle.c) -- CPU only.

Each test ties the oracle to something other than itself: the paper's printed
values, SPEC.md's worked examples, closed forms, an independently structured
formula (Eq. 5 with the corrected product index), the clamped-affine monoid,
invariants, and brute force on tiny inputs.  A plausible mistake in the oracle
(a dropped term, a wrong sign or index, add/decay swapped, a missing clamp,
wrong rounding) fails at least one of them; see DESIGN.md section 3.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import Oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def ev(rows):
    """rows: list of (t, x, y, p) -> structured array."""
    a = np.zeros(len(rows), dtype=[("t", "<i8"), ("x", "<u2"), ("y", "<u2"), ("p", "i1")])
    for i, r in enumerate(rows):
        a[i] = r
    return a


def eq5_weights_S(times, pols, C, k, b, T_init=0):
    """Eq. 5 with the product index read as j=i..n (
    DESIGN reading A2): S_n = C * sum_i p_i * prod_{j=i}^{n} d(t_j - t_{j-1}),
    t_0 = T_init.  Written with explicit products, no recursion."""
    n = len(times)
    tt = [T_init] + list(times)
    S = 0.0
    for i in range(1, n + 1):
        w = 1.0
        for j in range(i, n + 1):
            u = 1.0 - k * ((tt[j] - tt[j - 1]) / 1e6)
            w *= u ** b if u > 0 else 0.0
        S += pols[i - 1] * w
    return C * S


# ---------------------------------------------------------------- P1: SPEC examples
def test_spec_worked_examples():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for e in g["decay_factor"]:
        assert oracle.decay(e["dt_us"], e["k"], e["b"]) == pytest.approx(e["expect"], abs=1e-15), e
    for e in g["apply_event"]:
        o = Oracle(1, 1, C=e["C"], k=e["k"], b=e["b"], s_min=-1.5, s_max=1.5)
        if e["S0"] is not None:
            o.set_state(np.array([e["S0"]]), np.array([e["T0"]]))
        t, p = e["event"]
        assert o.push(ev([(t, 0, 0, p)])) == 0
        o.flush()
        S, T = o.get_state()
        assert S[0, 0] == pytest.approx(e["expect_S"], abs=1e-15), e
        assert T[0, 0] == e["expect_T"]
    for e in g["peek_decayed"]:
        o = Oracle(1, 1, k=e["k"], b=e["b"], s_min=-1.5, s_max=1.5)
        o.set_state(np.array([e["S0"]]), np.array([e["T0"]]))
        # the frame value is the peeked value mapped by Eq. 14
        fr = o.render(e["t_now"])
        assert fr[0, 0] == oracle.map_gray(e["expect"], -1.5, 1.5)
        S, T = o.get_state()           # peek does not mutate
        assert S[0, 0] == e["S0"] and T[0, 0] == e["T0"]
    for e in g["clamp"]:
        assert oracle.clamp(e["v"], e["lo"], e["hi"]) == e["expect"]
    for e in g["map_to_gray"]:
        assert oracle.map_gray(e["v"], e["lo"], e["hi"]) == e["expect"]


def test_spec_process_events_examples():
    # S:191 empty 30 ms at 100 FPS -> 3 uniform frames of 128
    o = Oracle(5, 4)
    fr = o.render_many([10000, 20000, 30000])
    assert fr.shape == (3, 4, 5) and (fr == 128).all()
    # S:192 one +1 event then silence (k=10, b=2): non-increasing toward 128.
    # The event arrives 10 ms after another one so it is not wiped by d(t-0).
    o = Oracle(1, 1, C=0.15, k=10, b=2)
    o.push(ev([(90000, 0, 0, 1), (100000, 0, 0, 1)]))
    vals = o.render_many([100000 + 10000 * i for i in range(12)])[:, 0, 0].astype(int)
    assert vals[0] > 128
    assert all(vals[i] >= vals[i + 1] for i in range(len(vals) - 1))
    assert vals[-1] == 128
    # S:193 hot pixel +1 at 10 kHz for 1 s saturates at 255 and never exceeds s_max
    o = Oracle(1, 1, C=0.15, k=10, b=2)
    o.push(ev([(100 * i, 0, 0, 1) for i in range(1, 10001)]))
    fr = o.render_many([100 * i for i in range(1000, 10001, 1000)])
    S, _ = o.get_state()
    assert S[0, 0] == 1.5 and (fr == 255).all()


# ---------------------------------------------------------------- P2: geometric closed form
def test_geometric_closed_form():
    C, k, b, D = 0.15, 10.0, 2.0, 10000
    rows = [r.split() for r in open(os.path.join(GOLD, "geometric_closed_form.txt")) if r[0] != "#"]
    o = Oracle(1, 1, C=C, k=k, b=b, s_min=-1.5, s_max=1.5)
    n_max = 200
    o.push(ev([(D * i, 0, 0, 1) for i in range(1, n_max + 1)]))
    frames = o.render_many([D * i for i in range(1, n_max + 1)])
    d = 0.81
    o2 = Oracle(1, 1, C=C, k=k, b=b, s_min=-1.5, s_max=1.5)
    for n in range(1, n_max + 1):
        o2.push(ev([(D * n, 0, 0, 1)]))
        o2.flush()
        S = o2.get_state()[0][0, 0]
        assert S == pytest.approx(C * d * (1 - d ** n) / (1 - d), abs=1e-13, rel=1e-12)
        # frame at t_f = t_n reads S_n undecayed (dt = 0), Eq. 14
        q = 255.0 * (S + 1.5) / 3.0
        assert frames[n - 1, 0, 0] == math.floor(q + 0.5)
    for n_str, val in rows:
        o3 = Oracle(1, 1, C=C, k=k, b=b)
        o3.push(ev([(D * i, 0, 0, 1) for i in range(1, int(n_str) + 1)]))
        o3.flush()
        assert o3.get_state()[0][0, 0] == pytest.approx(float(val), abs=1e-12)
    # limit: S_inf = C d / (1 - d)
    assert S == pytest.approx(C * d / (1 - d), abs=1e-12)


# ---------------------------------------------------------------- P3: Eq. 5 brute force
def test_eq5_brute_force_random_streams():
    rng = np.random.default_rng(3)
    for trial in range(100):
        n = int(rng.integers(1, 1001))
        k = float(rng.choice([10.0, 3.0, 100.0]))
        b = float(rng.choice([2.0, 1.0, 2.5, 0.5]))
        C = 0.15
        t = np.sort(rng.integers(0, 3_000_000, n)).astype(np.int64)
        x = rng.integers(0, 8, n).astype(np.uint16)
        y = rng.integers(0, 8, n).astype(np.uint16)
        p = rng.choice([-1, 1], n).astype(np.int8)
        o = Oracle(8, 8, C=C, k=k, b=b, s_min=-1e300, s_max=1e300)
        assert o.push((t, x, y, p)) == 0
        o.flush()
        S, T = o.get_state()
        for q in range(64):
            m = (y.astype(int) * 8 + x.astype(int)) == q
            if not m.any():
                assert S.flat[q] == 0.0 and T.flat[q] == 0
                continue
            ref = eq5_weights_S(list(t[m]), list(p[m].astype(int)), C, k, b)
            assert abs(S.flat[q] - ref) <= 1e-9, (trial, q)
            assert T.flat[q] == t[m][-1]


# ---------------------------------------------------------------- P4: baseline
@pytest.mark.parametrize("lo,hi", [(-1.5, 1.5), (-2.0, 1.0), (-0.3, 3.0), (0.5, 2.0)])
def test_baseline_uniform(lo, hi):
    o = Oracle(7, 3, s_min=lo, s_max=hi)
    fr = o.render(12345)
    v0 = min(max(0.0, lo), hi)
    expect = math.floor(255.0 * (v0 - lo) / (hi - lo) + 0.5)
    assert (fr == expect).all()


def test_decayed_pixel_returns_to_baseline_exactly():
    o = Oracle(2, 1, C=0.15, k=10, b=2)
    o.push(ev([(1000, 0, 0, 1), (2000, 0, 0, 1)]))
    fr = o.render_many([2000, 2000 + 99_999, 2000 + 100_000, 500_000])
    assert fr[0, 0, 0] > 128 and fr[1, 0, 0] == 128 and fr[2, 0, 0] == 128 and fr[3, 0, 0] == 128
    assert (fr[:, 0, 1] == 128).all()


# ---------------------------------------------------------------- P5: linearity / symmetry
def test_polarity_flip_negates_bit_exactly():
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = 500
        t = np.sort(rng.integers(0, 400_000, n)).astype(np.int64)
        x = rng.integers(0, 4, n).astype(np.uint16)
        y = rng.integers(0, 4, n).astype(np.uint16)
        p = rng.choice([-1, 1], n).astype(np.int8)
        fa, Sa, Ta = oracle.run(4, 4, (t, x, y, p), [400_000], s_min=-0.6, s_max=0.6)
        fb, Sb, Tb = oracle.run(4, 4, (t, x, y, -p), [400_000], s_min=-0.6, s_max=0.6)
        assert np.array_equal(Sa, -Sb) and np.array_equal(Ta, Tb)
        # floor(128 + a) + floor(128 - a) is 255 or 256 (Eq. 14 is symmetric about S=0)
        ssum = fa.astype(int) + fb.astype(int)
        assert ((ssum == 255) | (ssum == 256)).all()


def test_linearity_in_polarity_increments():
    # With the clamp disabled S is linear in the p_i (weights depend on times
    # only), so every mixed second difference vanishes.
    rng = np.random.default_rng(6)
    n = 300
    t = np.sort(rng.integers(0, 300_000, n)).astype(np.int64)
    x = np.zeros(n, np.uint16); y = np.zeros(n, np.uint16)
    p = rng.choice([-1, 1], n).astype(np.int8)

    def S_of(pp):
        _, S, _ = oracle.run(1, 1, (t, x, y, pp), [300_000], s_min=-1e300, s_max=1e300)
        return S[0, 0]
    base = S_of(p)
    for _ in range(20):
        i, j = rng.choice(n, 2, replace=False)
        pi = p.copy(); pi[i] = -pi[i]
        pj = p.copy(); pj[j] = -pj[j]
        pij = pi.copy(); pij[j] = -pij[j]
        assert abs(base - S_of(pi) - S_of(pj) + S_of(pij)) < 1e-12
    assert abs(base + S_of(-p)) < 1e-15


# ---------------------------------------------------------------- P6: Eq. 2 limit
def test_eq2_limit_tiny_k():
    rng = np.random.default_rng(7)
    n = 2000
    t = np.sort(rng.integers(0, 10_000_000, n)).astype(np.int64)
    p = rng.choice([-1, 1], n).astype(np.int8)
    z = np.zeros(n, np.uint16)
    C, lo, hi = 0.2, -1.0, 1.4
    _, S, _ = oracle.run(1, 1, (t, z, z, p), [10_000_000], C=C, k=1e-9, b=2, s_min=lo, s_max=hi)
    s = 0.0
    for pi in p:                       # Eq. 2 running sum with the Eq. 13 clamp
        s = min(max(s + int(pi) * C, lo), hi)
    assert abs(S[0, 0] - s) < 1e-9


# ---------------------------------------------------------------- P7/P8: saturation and cutoff
def test_hot_pixel_saturation_and_late_readout():
    o = Oracle(1, 1, C=0.15, k=10, b=2)
    o.push(ev([(100 * i, 0, 0, 1) for i in range(1, 101)]))
    fr = o.render(100 * 100 + 100)
    S, T = o.get_state()
    assert S[0, 0] == 1.5 and T[0, 0] == 10000
    # readout 100 us later: 1.5 * 0.999^2 = 1.4970015 -> 254.745 -> 255
    assert fr[0, 0] == 255


def test_cutoff_gap_zeroes_state():
    for b in (0.5, 1.0, 2.0, 3.3):
        o = Oracle(1, 1, C=0.15, k=10, b=b)
        o.push(ev([(50_000, 0, 0, 1), (150_000, 0, 0, 1)]))
        o.flush()
        assert o.get_state()[0][0, 0] == 0.0


# ---------------------------------------------------------------- P9: Eq. 6 property
def test_eq6_inequality_and_exponential_negative_control():
    rng = np.random.default_rng(9)
    for _ in range(10000):
        k = float(10 ** rng.uniform(-1, 2))
        b = float(10 ** rng.uniform(-1, 1))
        n = int(rng.integers(2, 11))
        horizon_us = 1e6 / (n * k)
        t_us = int(rng.uniform(0.05, 0.95) * horizon_us)
        if t_us < 1:
            continue
        lhs = oracle.decay(t_us, k, b) ** n
        rhs = oracle.decay(n * t_us, k, b)
        assert lhs > rhs, (k, b, n, t_us)
    # negative control: exponential decay compounds exactly
    for _ in range(1000):
        lam, a, c = rng.uniform(0.1, 50), rng.uniform(0, 1), rng.uniform(0, 1)
        assert abs(math.exp(-lam * a) * math.exp(-lam * c) - math.exp(-lam * (a + c))) < 1e-12


# ---------------------------------------------------------------- P10/P11: invariances
def _random_stream(rng, W, H, n, span):
    t = np.sort(rng.integers(0, span, n)).astype(np.int64)
    # clustered pixels so that many events share a pixel within 1/k
    x = (rng.integers(0, W, n) // 2 * 2).astype(np.uint16)
    y = rng.integers(0, H, n).astype(np.uint16)
    p = rng.choice([-1, 1], n).astype(np.int8)
    return t, x, y, p


def test_frame_rate_independence_of_state():
    rng = np.random.default_rng(10)
    t, x, y, p = _random_stream(rng, 6, 5, 20000, 1_000_000)
    states = []
    for fps in (10, 100, 1000):
        period = 1_000_000 // fps
        _, S, T = oracle.run(6, 5, (t, x, y, p), np.arange(1, fps + 1) * period)
        states.append((S, T))
    for S, T in states[1:]:
        assert np.array_equal(S, states[0][0]) and np.array_equal(T, states[0][1])


def test_batch_split_invariance():
    rng = np.random.default_rng(11)
    t, x, y, p = _random_stream(rng, 5, 5, 5000, 500_000)
    tf = np.arange(1, 51) * 10_000
    f0, S0, T0 = oracle.run(5, 5, (t, x, y, p), tf)
    for _ in range(5):
        cuts = sorted(rng.choice(len(t), 3, replace=False))
        o = Oracle(5, 5)
        prev = 0
        for c in list(cuts) + [len(t)]:
            assert o.push((t[prev:c], x[prev:c], y[prev:c], p[prev:c])) == 0
            prev = c
        f1 = o.render_many(tf)
        S1, T1 = o.get_state()
        assert np.array_equal(f0, f1) and np.array_equal(S0, S1) and np.array_equal(T0, T1)
    # interleaving pushes with renders gives the same frames too
    o = Oracle(5, 5)
    outs = []
    for j, tfj in enumerate(tf):
        m = (t > (tf[j - 1] if j else -1)) & (t <= tfj)
        o.push((t[m], x[m], y[m], p[m]))
        outs.append(o.render(tfj))
    assert np.array_equal(np.stack(outs), f0)


# ---------------------------------------------------------------- P12/P13: monoid + tiny brute force
def compose(f, g):
    """g after f for maps s -> clamp(a*s + c, lo, hi) with a >= 0."""
    a1, c1, lo1, hi1 = f
    a2, c2, lo2, hi2 = g
    cl = lambda v: min(max(v, lo2), hi2)
    return (a2 * a1, a2 * c1 + c2, cl(a2 * lo1 + c2), cl(a2 * hi1 + c2))


def apply_map(f, s):
    a, c, lo, hi = f
    return min(max(a * s + c, lo), hi)


def event_map(dt_us, p, C, k, b, lo, hi):
    d = oracle.decay(dt_us, k, b)
    return (d, d * p * C, lo, hi)


def test_monoid_composition_matches_oracle():
    rng = np.random.default_rng(12)
    C, k, b, lo, hi = 0.15, 10.0, 2.0, -0.5, 0.7
    for _ in range(200):
        n = int(rng.integers(1, 60))
        t = np.sort(rng.integers(0, 200_000, n)).astype(np.int64)
        p = rng.choice([-1, 1], n).astype(np.int8)
        z = np.zeros(n, np.uint16)
        _, S, T = oracle.run(1, 1, (t, z, z, p), [200_000], C=C, k=k, b=b, s_min=lo, s_max=hi)
        F = (1.0, 0.0, -1e308, 1e308)   # identity map
        prev = 0
        for ti, pi in zip(t, p):
            F = compose(F, event_map(int(ti) - prev, int(pi), C, k, b, lo, hi))
            prev = int(ti)
        assert abs(apply_map(F, 0.0) - S[0, 0]) < 1e-12
    # associativity on random maps
    for _ in range(2000):
        fs = [(rng.uniform(0, 1), rng.uniform(-1, 1), -rng.uniform(0, 2), rng.uniform(0, 2)) for _ in range(3)]
        A = compose(compose(fs[0], fs[1]), fs[2])
        B = compose(fs[0], compose(fs[1], fs[2]))
        assert all(abs(u - v) < 1e-12 for u, v in zip(A, B))


def test_tiny_brute_force_three_way():
    C, k, b = 0.15, 10.0, 2.0
    times = [0, 1, 2, 10000, 99999, 100000, 100001]
    clamps = [(-1e300, 1e300), (-0.2, 0.2), (-0.1, 0.25)]
    checked = 0
    for n in range(1, 5):
        for ts in itertools.combinations_with_replacement(times, n):
            for ps in itertools.product([-1, 1], repeat=n):
                for pixs in itertools.product([0, 1], repeat=n):
                    if n == 4 and (pixs[0] == 1 or ps[0] == -1):
                        continue   # keep the enumeration a few seconds long
                    t = np.array(ts, np.int64); p = np.array(ps, np.int8)
                    x = np.array(pixs, np.uint16); y = np.zeros(n, np.uint16)
                    for lo, hi in clamps:
                        _, S, T = oracle.run(2, 1, (t, x, y, p), [ts[-1]], C=C, k=k, b=b,
                                             s_min=lo, s_max=hi)
                        for q in (0, 1):
                            m = x == q
                            F = (1.0, 0.0, -1e308, 1e308)   # identity map
                            prev = 0
                            for ti, pi in zip(t[m], p[m]):
                                F = compose(F, event_map(int(ti) - prev, int(pi), C, k, b, lo, hi))
                                prev = int(ti)
                            assert abs(apply_map(F, 0.0) - S[0, q]) < 1e-12
                            if lo < -1e299:
                                ref = eq5_weights_S(list(t[m]), list(p[m].astype(int)), C, k, b) if m.any() else 0.0
                                assert abs(ref - S[0, q]) < 1e-12
                            checked += 1
    assert checked > 10000


# ---------------------------------------------------------------- P14: stable grouping definition
def test_stable_group_by_is_stable_sort():
    rng = np.random.default_rng(14)
    for _ in range(50):
        keys = rng.integers(0, 17, 400)
        perm = oracle.stable_group_by(keys)
        ref = sorted(range(len(keys)), key=lambda i: keys[i])   # Python sort is stable
        assert list(perm) == ref


# ---------------------------------------------------------------- P15: the paper's printed numbers
def test_fig4_printed_values_pin_15_percent_reading():
    rows = [r.split() for r in open(os.path.join(GOLD, "fig4_threshold.txt")) if r[0] != "#"]
    c = math.log(1.15)            # reading A12: a 15 % threshold is ln(1.15) in log units
    for ratio, printed, tol in rows:
        n_events = math.log(float(ratio)) / c       # events needed for the ratio
        assert abs(math.log(1 + n_events) - float(printed)) <= float(tol)
    # the other reading (c = 0.15) would print 1.73 / 2.12
    assert abs(math.log(1 + math.log(2) / 0.15) - 1.8) > 0.05


# ---------------------------------------------------------------- Alg. 2 literal readout and errors
def test_readout_decay_off_is_alg2_literal():
    o = Oracle(1, 1, C=0.15, k=10, b=2, readout_decay=0)
    o.push(ev([(90000, 0, 0, 1), (100000, 0, 0, 1)]))
    fr = o.render_many([100000, 150000, 1_000_000])
    S, _ = o.get_state()
    assert (fr[:, 0, 0] == oracle.map_gray(S[0, 0], -1.5, 1.5)).all()


def test_validation_errors_and_atomic_push():
    o = Oracle(4, 3)
    assert o.push(ev([(5, 4, 0, 1)])) == oracle.ESIO_ERR_OUT_OF_BOUNDS
    assert o.push(ev([(5, 0, 3, 1)])) == oracle.ESIO_ERR_OUT_OF_BOUNDS
    assert o.push(ev([(5, 1, 1, 0)])) == oracle.ESIO_ERR_BAD_POLARITY
    assert o.push(ev([(5, 1, 1, 1), (4, 1, 1, 1)])) == oracle.ESIO_ERR_NEGATIVE_INTERVAL
    assert o.pending() == 0                        # atomic: nothing kept
    assert o.push(ev([(5, 1, 1, 1), (5, 1, 1, -1)])) == 0
    o.render(10)
    assert o.push(ev([(10, 1, 1, 1)])) == oracle.ESIO_ERR_NEGATIVE_INTERVAL   # <= last frame
    assert o.push(ev([(11, 1, 1, 1)])) == 0
    with pytest.raises(oracle.OracleError):
        o.render(9)                                # frames must not go back in time


def test_pure_python_copy_agrees_on_small_inputs():
    rng = np.random.default_rng(15)
    for b in (2.0, 0.5):
        t, x, y, p = _random_stream(rng, 6, 4, 3000, 300_000)
        tf = np.arange(1, 31) * 10_000
        f0, S0, T0 = oracle.run(6, 4, (t, x, y, p), tf, b=b, s_min=-0.4, s_max=0.5)
        f1, S1, T1 = oracle.py_run(6, 4, (t, x, y, p), tf, b=b, s_min=-0.4, s_max=0.5)
        assert np.array_equal(f0, f1) and np.array_equal(T0, T1)
        assert np.max(np.abs(S0 - S1)) < 1e-12


# ---------------------------------------------------------------- P14: decay variants
def test_exp_decay_spec_examples_and_exponent_law():
    """SPEC S:261-263 (expdecay_process examples): dt = 0 -> 1; lambda = 10,
    dt = 0.1 s -> e^-1; n-step compounding equals one long decay (the
    structural contrast to ESI's Eq. 6)."""
    L = oracle.lib()
    assert L.esio_decay_exp(0, 10.0) == 1.0
    assert L.esio_decay_exp(100_000, 10.0) == pytest.approx(math.exp(-1.0), rel=1e-15)
    rng = np.random.default_rng(21)
    for _ in range(2000):
        lam = float(rng.uniform(0.1, 50))
        a, c = int(rng.integers(0, 200_000)), int(rng.integers(0, 200_000))
        assert abs(L.esio_decay_exp(a, lam) * L.esio_decay_exp(c, lam) - L.esio_decay_exp(a + c, lam)) < 1e-12
        n = int(rng.integers(2, 9))
        assert L.esio_decay_exp(a, lam) ** n == pytest.approx(L.esio_decay_exp(n * a, lam), rel=1e-12)


def test_complementary_filter_spec_example():
    """alpha = 5, two +1 events 0.2 s apart, C = 0.15, decay then add
    -> 0.15 e^-1 + 0.15 = 0.2052 (exp decay, decay_first)."""
    o = Oracle(1, 1, C=0.15, k=5.0, b=2.0, s_min=-1.5, s_max=1.5, decay_kind=1, decay_first=1)
    o.push(ev([(1_000_000, 0, 0, 1), (1_200_000, 0, 0, 1)]))
    o.flush()
    S = o.get_state()[0][0, 0]
    assert S == pytest.approx(0.15 * math.exp(-1.0) + 0.15, rel=1e-14)
    assert round(S, 4) == 0.2052
    # a single +1 event -> value C at the event time
    o2 = Oracle(1, 1, C=0.15, k=5.0, decay_kind=1, decay_first=1)
    o2.push(ev([(300_000, 0, 0, 1)]))
    assert o2.render(300_000)[0] == math.floor(255 * (0.15 + 1.5) / 3.0 + 0.5)
    o2.flush()
    assert o2.get_state()[0][0, 0] == 0.15


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("first", [0, 1])
def test_variant_geometric_closed_forms(kind, first):
    """Evenly spaced (D) same-polarity events from the origin, q = d(D):
    add-then-decay (Alg. 2): S_n = C q (1 - q^n) / (1 - q);
    decay-then-add:          S_n = C (1 - q^n) / (1 - q)
    (sums of a geometric series; q = (1 - kD)^b or e^{-kD})."""
    C, k, b, D = 0.15, 10.0, 2.0, 10_000
    q = math.exp(-k * D / 1e6) if kind else (1 - k * D / 1e6) ** b
    o = Oracle(1, 1, C=C, k=k, b=b, s_min=-5.0, s_max=5.0, decay_kind=kind, decay_first=first)
    for n in range(1, 120):
        o.push(ev([(D * n, 0, 0, 1)]))
        o.flush()
        S = o.get_state()[0][0, 0]
        want = C * (1 - q ** n) / (1 - q) * (1.0 if first else q)
        assert S == pytest.approx(want, rel=1e-12, abs=1e-14), (n, S, want)


def test_esi_decay_first_two_events():
    """Eq. 4 decay then add, two +1 events 0.05 s apart at k = 10, b = 2:
    S = C (1 - 0.5)^2 + C = 1.25 C (first event: 0 * d + C)."""
    o = Oracle(1, 1, C=0.15, k=10.0, b=2.0, decay_first=1)
    o.push(ev([(20_000, 0, 0, 1), (70_000, 0, 0, 1)]))
    o.flush()
    assert o.get_state()[0][0, 0] == pytest.approx(0.15 * 1.25, rel=1e-15)


@pytest.mark.parametrize("kind,first", [(1, 0), (0, 1), (1, 1)])
def test_variant_pure_python_copy_agrees(kind, first):
    rng = np.random.default_rng(30 + 2 * kind + first)
    t, x, y, p = _random_stream(rng, 6, 4, 3000, 300_000)
    tf = np.arange(1, 31) * 10_000
    f0, S0, T0 = oracle.run(6, 4, (t, x, y, p), tf, s_min=-0.4, s_max=0.5, decay_kind=kind, decay_first=first)
    f1, S1, T1 = oracle.py_run(6, 4, (t, x, y, p), tf, s_min=-0.4, s_max=0.5, decay_kind=kind, decay_first=first)
    assert np.array_equal(f0, f1) and np.array_equal(T0, T1)
    assert np.max(np.abs(S0 - S1)) < 1e-12


# ---------------------------------------------------------------- P15: Eq. 2 naive integrator
def test_naive_integrator_spec_examples_and_pathology():
    """SPEC S:253-255 (naive_process): +1 then -1 cancel exactly; n equal
    events give n C; on a pure-noise stream |S| at the worst pixel leaves any
    fixed bound (random walk, the Fig. 4 pathology) while ESI's state
    stays inside [S_min, S_max]; frames clamp at render time."""
    o = Oracle(1, 1, C=0.15, decay_kind=2)
    o.push(ev([(10, 0, 0, 1), (20, 0, 0, -1)]))
    o.flush()
    assert o.get_state()[0][0, 0] == 0.0
    o2 = Oracle(1, 1, C=0.15, decay_kind=2)
    o2.push(ev([(10 * i, 0, 0, 1) for i in range(1, 41)]))
    o2.flush()
    assert o2.get_state()[0][0, 0] == pytest.approx(40 * 0.15, rel=1e-14)    # 6.0 > S_max: no clamp
    assert o2.render(1_000_000)[0] == 255                                    # clamped at render
    rng = np.random.default_rng(40)
    n = 200_000
    t = np.sort(rng.integers(0, 20_000_000, n)).astype(np.int64)
    x = rng.integers(0, 4, n).astype(np.uint16)
    y = np.zeros(n, np.uint16)
    p = rng.choice([-1, 1], n).astype(np.int8)
    _, Sn, _ = oracle.run(4, 1, (t, x, y, p), [20_000_000], decay_kind=2)
    _, Se, _ = oracle.run(4, 1, (t, x, y, p), [20_000_000])
    assert np.abs(Sn).max() > 1.5 and np.abs(Se).max() <= 1.5
    # the naive state is exactly C * (sum of polarities) per pixel
    for q in range(4):
        assert Sn[0, q] == pytest.approx(0.15 * int(p[x == q].astype(np.int64).sum()), abs=1e-9)


def test_naive_pure_python_copy_agrees():
    rng = np.random.default_rng(41)
    t, x, y, p = _random_stream(rng, 6, 4, 3000, 300_000)
    tf = np.arange(1, 31) * 10_000
    f0, S0, T0 = oracle.run(6, 4, (t, x, y, p), tf, s_min=-0.4, s_max=0.5, decay_kind=2)
    f1, S1, T1 = oracle.py_run(6, 4, (t, x, y, p), tf, s_min=-0.4, s_max=0.5, decay_kind=2)
    assert np.array_equal(f0, f1) and np.array_equal(T0, T1)
    assert np.max(np.abs(S0 - S1)) < 1e-12


def test_complementary_filter_unclamped_state():
    """Events-only complementary filter: exp decay,
    decay then add, no per-event clamp, frames clamp at render.  Two +1 events
    0.2 s apart at alpha = 5 give 0.2052 even with S_max = 0.2; the clamped
    variant stops at 0.2; the frame is 255 either way; long silence relaxes the
    frame to the baseline gray."""
    kw = dict(C=0.15, k=5.0, s_min=-0.2, s_max=0.2, decay_kind=1, decay_first=1)
    evs = ev([(1_000_000, 0, 0, 1), (1_200_000, 0, 0, 1)])
    o = Oracle(1, 1, state_unclamped=1, **kw)
    o.push(evs)
    assert o.render(1_200_000)[0] == 255
    assert o.get_state()[0][0, 0] == pytest.approx(0.15 * math.exp(-1.0) + 0.15, rel=1e-14)
    assert o.render(20_000_000)[0] == 128                       # 18.8 s at alpha = 5: e^-94 -> mid-gray
    o2 = Oracle(1, 1, **kw)
    o2.push(evs)
    o2.flush()
    assert o2.get_state()[0][0, 0] == 0.2
    rng = np.random.default_rng(42)
    t, x, y, p = _random_stream(rng, 6, 4, 3000, 300_000)
    tf = np.arange(1, 31) * 10_000
    f0, S0, T0 = oracle.run(6, 4, (t, x, y, p), tf, state_unclamped=1, **kw)
    f1, S1, T1 = oracle.py_run(6, 4, (t, x, y, p), tf, state_unclamped=1, **kw)
    assert np.array_equal(f0, f1) and np.max(np.abs(S0 - S1)) < 1e-12
    assert np.abs(S0).max() > 0.2                                # the state does leave the bounds


# ---------------------------------------------------------------- A8: Eq. 14 rounding (SPEC acceptance 9)
def test_eq14_exact_ties_round_half_away():
    """Exact ties of the Eq. 14 argument round half away from zero
    (reading A8).  Hand-rounded values in
    golden/eq14_ties.json; a half-to-even rounding (rint) fails here."""
    g = json.load(open(os.path.join(GOLD, "eq14_ties.json")))
    for c in g["cases"]:
        assert oracle.map_gray(c["v"], c["lo"], c["hi"]) == c["expect"], c


def test_eq14_all_256_gray_levels_randomized_bounds():
    """SPEC acceptance 9: endpoints map to 0/255, the mid value maps to
    128, and every target gray level g is reached, exhaustively over all 256
    levels with randomized bounds.  Bounds are [lo, lo + 255 h] with h a power
    of two and lo a multiple of h, so v = lo + g h gives the Eq. 14 argument g
    exactly and v = lo + (g + 1/2) h gives the exact tie g + 1/2, which the
    stated rule (half away from zero) sends to g + 1."""
    rng = np.random.default_rng(540)
    for _ in range(40):
        h = 2.0 ** int(rng.integers(-10, 5))
        lo = float(rng.integers(-300, 40)) * h
        hi = lo + 255.0 * h
        assert oracle.map_gray(lo, lo, hi) == 0 and oracle.map_gray(hi, lo, hi) == 255
        assert oracle.map_gray(lo + 127.5 * h, lo, hi) == 128          # mid value
        for gl in range(256):
            assert oracle.map_gray(lo + gl * h, lo, hi) == gl
            if gl < 255:
                assert oracle.map_gray(lo + (gl + 0.5) * h, lo, hi) == gl + 1
                # just below / above the tie (h/1024, exact) stay on their side
                below = lo + (gl + 0.5 - 1 / 1024) * h
                above = lo + (gl + 0.5 + 1 / 1024) * h
                assert oracle.map_gray(below, lo, hi) == gl
                assert oracle.map_gray(above, lo, hi) == gl + 1
        # clamp contracts: idempotent and monotone
        vs = np.sort(rng.uniform(lo - 10 * h, hi + 10 * h, 64))
        cl = [oracle.clamp(v, lo, hi) for v in vs]
        assert all(oracle.clamp(c, lo, hi) == c for c in cl)
        assert all(a <= b for a, b in zip(cl, cl[1:]))
        gray = [oracle.map_gray(c, lo, hi) for c in cl]
        assert all(a <= b for a, b in zip(gray, gray[1:]))


def test_eq14_ties_through_the_render_path():
    """The frame bytes of a render carry the same rounding: state values on
    exact ties (Alg. 2 literal readout) give the half-away bytes."""
    g = json.load(open(os.path.join(GOLD, "eq14_ties.json")))
    for c in g["cases"]:
        if not (c["lo"] <= 0.0 <= c["hi"]) or c["lo"] == c["hi"]:
            continue
        o = Oracle(1, 1, s_min=c["lo"], s_max=c["hi"], readout_decay=0)
        o.set_state(np.array([c["v"]]), np.array([0]))
        assert o.render(10)[0, 0] == c["expect"], c


# ---------------------------------------------------------------- SPEC metrics, f3
def test_metrics_pins():
    """SPEC score_frame examples and the affine-invariance property
    (S:425): recon = a x + b (a > 0) -> pearson 1, mse_norm 0; negated -> -1, 4;
    uniform recon -> missing; mse_norm = 2 (1 - pearson) for any pair."""
    from oracle.metrics import score_frame, score_run
    rng = np.random.default_rng(401)
    truth = rng.normal(size=(24, 32))
    for _ in range(20):
        a, b = rng.uniform(0.01, 50), rng.uniform(-100, 100)
        r, m = score_frame(a * truth + b, truth)
        assert abs(r - 1.0) <= 1e-9 and abs(m) <= 1e-9
        r, m = score_frame(-a * truth + b, truth)
        assert abs(r + 1.0) <= 1e-9 and abs(m - 4.0) <= 1e-8
    r, m = score_frame(np.full((24, 32), 128), truth)
    assert np.isnan(r) and np.isnan(m)
    x = rng.normal(size=(24, 32))
    r, m = score_frame(x, truth)
    assert abs(m - 2 * (1 - r)) <= 1e-12
    assert abs(r - np.corrcoef(x.ravel(), truth.ravel())[0, 1]) <= 1e-12    # textbook definition
    sc, summ = score_run([x, np.zeros((24, 32)), truth], [truth] * 3)
    assert summ["missing"] == 1 and abs(summ["min"] - r) <= 1e-12
    assert abs(summ["mean"] - (r + 1.0) / 2) <= 1e-12


# ---------------------------------------------------------------- SPEC acceptance 4, Fig. 4
def _noise_stream(seed, W=128, H=128, rate=5.0, dur_us=2_000_000, hot=(64, 64), hot_hz=10_000.0):
    """SPEC acceptance 4: a 2 s pure-noise stream, background 5 ev/px/s (Poisson,
    random polarity), one hot pixel at 10 kHz (Fig. 3: noise events and a hot
    pixel)."""
    rng = np.random.default_rng(seed)
    n_bg = rng.poisson(rate * W * H * dur_us * 1e-6)
    n_hot = rng.poisson(hot_hz * dur_us * 1e-6)
    t = np.concatenate([rng.integers(0, dur_us, n_bg), rng.integers(0, dur_us, n_hot)])
    x = np.concatenate([rng.integers(0, W, n_bg), np.full(n_hot, hot[0])])
    y = np.concatenate([rng.integers(0, H, n_bg), np.full(n_hot, hot[1])])
    p = rng.choice(np.array([-1, 1], np.int8), n_bg + n_hot)
    o = np.argsort(t, kind="stable")
    a = np.zeros(len(t), dtype=[("t", "<i8"), ("x", "<u2"), ("y", "<u2"), ("p", "i1")])
    a["t"], a["x"], a["y"], a["p"] = t[o], x[o], y[o], p[o]
    return a


def test_fig4_noise_pathology_factor_oracle():
    """SPEC acceptance 4 (Fig. 4 'severe noise will quickly
    destroy the estimated intensity'): on the pure-noise stream the naive Eq. 2
    integrator's 99th-percentile |S| exceeds ESI's (pre-clamp: the per-event
    clamp removed) by a factor >= 5, and ESI's clamped state stays inside
    [s_min, s_max].  Monte-Carlo confirmation of the constant: the
    factor on five seeds is printed by the assertion message."""
    W = H = 128
    tf = [2_000_000]
    facs = []
    for seed in range(5):
        a = _noise_stream(4000 + seed)
        _, S_naive, _ = oracle.run(W, H, a, tf, decay_kind=2)
        _, S_pre, _ = oracle.run(W, H, a, tf, state_unclamped=1)
        _, S_esi, _ = oracle.run(W, H, a, tf)
        facs.append(np.percentile(np.abs(S_naive), 99) / np.percentile(np.abs(S_pre), 99))
        assert S_esi.min() >= -1.5 and S_esi.max() <= 1.5
    assert min(facs) >= 5.0, facs
