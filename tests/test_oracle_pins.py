"""Pins for the CPU oracle (oracle/spice_oracle.c) against what the paper and the
mathematics fix — never against the oracle itself.  CPU only (``-m "not gpu"``).

Each test names the passage / reading it follows.
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.stats as st

import workloads as W
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cfg(model, n, n_exc, rules, params, delay=1, seed=3, activity=0.0, dt=0.1):
    return W.NetConfig("t", model, n, n_exc, tuple(rules), dt, delay, seed, activity, tuple(params))


def _brunel_params(**kw):
    p = dict(tau=20.0, VL=0.0, theta=20.0, Vr=10.0, tref=2.0, JE=0.1, g=5.0, lam=0.0, vlo=0.0, vhi=20.0)
    p.update(kw)
    return (p["tau"], p["VL"], p["theta"], p["Vr"], p["tref"], p["JE"], p["g"], p["lam"], p["vlo"], p["vhi"])


# --------------------------------------------------------------------------- RNG
def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox_kat.txt; reading R9)."""
    n = 0
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        assert list(O.philox(w[0:4], w[4:6])) == w[6:10]
        n += 1
    assert n == 3


# --------------------------------------------------------------------- partition
def test_partition_fig4_and_pigeonhole():
    """Fig. 4 alternating slices; SPEC S:368 pigeonhole counts."""
    for line in open(os.path.join(GOLD, "partition.txt")):
        if line.startswith("#") or not line.strip():
            continue
        head, ids = line.split(":")
        N, G, S, g = map(int, head.split())
        owned = [j for j in range(N) if O.owner(j, G, S) == g]
        assert owned == list(map(int, ids.split()))
        # Listing 1 enumerates exactly the owned set, ascending, stopping at j >= N
        listing = []
        i = 0
        while True:
            j = O.local_to_global(i, g, G, S)
            if j >= N:
                break
            listing.append(j)
            i += 1
        assert listing == owned


def test_listing1_worked_values():
    for line in open(os.path.join(GOLD, "listing1.txt")):
        if line.startswith("#") or not line.strip():
            continue
        S, G, g, i, j = map(int, line.split())
        assert O.local_to_global(i, g, G, S) == j


@pytest.mark.parametrize("N,G,S", [(1000, 3, 32), (4097, 8, 32), (100, 1, 7), (10, 4, 1)])
def test_partition_covers_and_balances(N, G, S):
    own = np.array([O.owner(j, G, S) for j in range(N)])
    counts = np.bincount(own, minlength=G)
    assert counts.sum() == N
    assert counts.max() - counts.min() <= S          # SPEC S:218 pigeonhole
    assert all(O.local_to_global(i, 0, 1, S) == i for i in range(50))  # G=1 identity


# ------------------------------------------------------------------ connectivity
def test_fig1_row_split():
    """Fig. 1: row {1,3,5,6,7,9} split at pivot 4 -> {1,3} | {5,6,7,9}.
    Built from p=1 rules (complete sub-ranges), split through the ownership filter
    with G=2, S=5 (every target < 4 is < 5 and vice versa for this row)."""
    line = open(os.path.join(GOLD, "fig1_split.txt")).read().splitlines()[-1]
    row, pivot, left, right = [list(map(int, x.split())) for x in line.split("|")]
    rules = [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0), W.Rule((0, 1), (3, 4), W.FIXED_PROB, 1.0),
             W.Rule((0, 1), (5, 8), W.FIXED_PROB, 1.0), W.Rule((0, 1), (9, 10), W.FIXED_PROB, 1.0)]
    cfg = _cfg(W.BRUNEL, 10, 10, rules, _brunel_params())
    rp, tg = O.OracleNet(cfg).csr()
    assert list(tg[rp[0]:rp[1]]) == row
    halves = []
    for g in range(2):
        rp2, tg2 = O.OracleNet(cfg, part=(g, 2, 5)).csr()
        halves.append(list(tg2[rp2[0]:rp2[1]]))
    assert halves == [left, right] and pivot == [4]


def test_p0_and_p1_special_cases():
    cfg1 = _cfg(W.BRUNEL, 37, 30, [W.Rule((0, 37), (0, 37), W.FIXED_PROB, 1.0)], _brunel_params())
    rp, tg = O.OracleNet(cfg1).csr()
    assert all(list(tg[rp[s]:rp[s + 1]]) == list(range(37)) for s in range(37))
    cfg0 = _cfg(W.BRUNEL, 37, 30, [W.Rule((0, 37), (0, 37), W.FIXED_PROB, 0.0)], _brunel_params())
    assert O.OracleNet(cfg0).nnz == 0


def test_vogels_edge_count_and_sorted_rows():
    """E = sum |src||dst| p within 5 sigma (BASELINE configs[0]: ~320K synapses); rows
    sorted ascending."""
    cfg = W.vogels(4000)
    net = O.OracleNet(cfg)
    rp, tg = net.csr()
    p = 0.02
    mean = 4000 * 4000 * p
    sd = np.sqrt(mean * (1 - p))
    assert abs(net.nnz - mean) < 5 * sd
    for s in range(0, 4000, 97):
        row = tg[rp[s]:rp[s + 1]]
        assert np.all(np.diff(row.astype(np.int64)) > 0)   # fixed prob: strictly ascending


def test_fixed_prob_degree_distribution_and_width_bound():
    """Out- and in-degree ~ Binomial(|range2|, p); the width estimate
    mu + 3 sigma is exceeded by <= 0.5 % of rows (SPEC acceptance 3)."""
    n, p = 3000, 0.1
    cfg = _cfg(W.BRUNEL, n, n, [W.Rule((0, n), (0, n), W.FIXED_PROB, p)], _brunel_params(), seed=11)
    rp, tg = O.OracleNet(cfg).csr()
    outdeg = np.diff(rp.astype(np.int64))
    indeg = np.bincount(tg, minlength=n)
    mu, var = n * p, n * p * (1 - p)
    for deg in (outdeg, indeg):
        assert abs(deg.mean() - mu) < 5 * np.sqrt(var / n)
        assert abs(deg.var() - var) < 0.15 * var
        # chi-square against the binomial pmf on pooled bins
        edges = np.arange(int(mu - 3 * np.sqrt(var)), int(mu + 3 * np.sqrt(var)) + 2)
        obs = np.histogram(deg, bins=np.concatenate(([-1], edges, [n + 1])))[0]
        cdf = st.binom.cdf(np.concatenate(([-1], edges, [n + 1])) - 1, n, p)
        exp = np.diff(cdf) * n
        keep = exp > 5
        chi2 = ((obs[keep] - exp[keep]) ** 2 / exp[keep]).sum()
        assert st.chi2.sf(chi2, keep.sum() - 1) > 1e-4
    width = mu + 3 * np.sqrt(var)
    assert (outdeg > width).mean() <= 0.005


def test_fixed_indegree_exact_count_and_uniform_sources():
    """Fixed in-degree rule (reading R9): exactly K edges per target, sources uniform."""
    n, k = 2000, 50
    cfg = W.synth(n, k, 0.005, seed=5)
    net = O.OracleNet(cfg)
    rp, tg = net.csr()
    assert net.nnz == n * k
    assert np.all(np.bincount(tg, minlength=n) == k)
    outdeg = np.diff(rp.astype(np.int64))
    chi2 = ((outdeg - k) ** 2 / k).sum()          # multinomial, expected k per source
    assert st.chi2.sf(chi2, n - 1) > 1e-4
    for s in range(0, n, 37):
        assert np.all(np.diff(tg[rp[s]:rp[s + 1]].astype(np.int64)) >= 0)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_partition_independence_union(G):
    """Each slice keeps exactly the edges whose target it owns; the union over ranks is
    the G=1 edge set ("the only data that need to be exchanged … are spikes";
    SPEC S:145)."""
    S = 32
    for cfg in (W.brunel(1500, 0.1, seed=4), W.synth(1200, 40, seed=9)):
        rp, tg = O.OracleNet(cfg).csr()
        rows_full = [tg[rp[s]:rp[s + 1]] for s in range(cfg.n)]
        parts = [O.OracleNet(cfg, part=(g, G, S)).csr() for g in range(G)]
        for s in range(cfg.n):
            merged = np.sort(np.concatenate([p[1][p[0][s]:p[0][s + 1]] for p in parts]))
            assert np.array_equal(merged, rows_full[s])
        for g, (rp2, tg2) in enumerate(parts):
            assert np.all((tg2 // S) % G == g)


# ------------------------------------------------------------------------ Poisson
@pytest.mark.parametrize("lam", [0.5, 2.0, 8.0, 16.0])
def test_poisson_table_against_scipy(lam):
    """External drive table (reading R12) vs the library CDF."""
    T = O.poisson_table(lam)
    assert T[-1] == 2 ** 32
    ks = np.arange(len(T) - 1)
    ref = np.floor(st.poisson.cdf(ks, lam) * 2.0 ** 32)
    assert np.all(np.abs(T[:-1].astype(np.float64) - ref) <= 4)
    assert st.poisson.sf(len(T) - 1, lam) < 2e-9


# ------------------------------------------------------------------- dynamics pins
def _one_neuron_brunel(precision, v0, **kw):
    cfg = _cfg(W.BRUNEL, 1, 1, [], _brunel_params(**kw))
    net = O.OracleNet(cfg, precision)
    net.set_state(O.F_V, np.array([v0]))
    return net


@pytest.mark.parametrize("precision,tol", [("ref64", 1e-12), ("mirror32", 1e-5)])
def test_lif_subthreshold_closed_form(precision, tol):
    """Forward Euler leak without input: V_k = V_L + (V0 - V_L)(1-h)^k exactly
    (reading R3).  Error measured against the span V0 - V_L = 20 mV (the trajectory
    crosses 0, so a pointwise relative error is meaningless there); fp32 rounding
    accumulates at most 3 * 2^-24 * 16 / h = 5.7e-4 mV, observed ~2e-6."""
    net = _one_neuron_brunel(precision, 15.0, VL=-5.0, theta=1e9)
    h = 0.1 / 20.0
    vs = []
    for _ in range(1000):
        net.step(1)
        vs.append(net.state(O.F_V)[0])
    k = np.arange(1, 1001)
    ref = -5.0 + 20.0 * (1 - h) ** k
    assert np.max(np.abs(np.array(vs, dtype=np.float64) - ref)) < tol * 20.0
    # and it is the Euler recurrence, not the exact exponential (-1.25 % at k = 1000)
    assert abs(vs[-1] - (-5 + 20 * np.exp(-h * 1000))) > 1e-3


@pytest.mark.parametrize("precision", ["ref64", "mirror32"])
def test_isi_constant_drive_closed_form(precision):
    """Reading R5 (reset, refractory): constant drive c = 0.15 mV/step (driver neuron 0
    forced every step, weight J_E = 0.15, delay 1), V_L=0, V_r=10, theta=20, h=0.005,
    R = 20: after a spike the neuron is held R steps, then V_k = 30 - 20 (1-h)^k first
    reaches theta at k = 139 (V = 20.0359; k = 138 gives 19.9858), so ISI = R + 139."""
    cfg = _cfg(W.BRUNEL, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0)],
               _brunel_params(JE=0.15, vlo=10.0, vhi=10.0))
    net = O.OracleNet(cfg, precision)
    for _ in range(1000):
        net.force_next([0], "add")
        net.step(1)
    t1 = [t for t, s in enumerate(net.spikes()) if 1 in s]
    isi = np.diff(t1)
    assert len(isi) >= 4 and np.all(isi == 20 + 139)


@pytest.mark.parametrize("precision", ["ref64", "mirror32"])
@pytest.mark.parametrize("gap,fires", [(80, True), (81, False), (1, True)])
def test_coincidence_window(precision, gap, fires):
    """Reading R6: two inputs of 12 mV into a neuron at rest (theta=20): it spikes iff
    12 (1-h)^gap + 12 >= 20, i.e. gap <= 80 (20.0358 at 80, 19.9956 at 81)."""
    cfg = _cfg(W.BRUNEL, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0)],
               _brunel_params(JE=12.0, vlo=0.0, vhi=0.0))
    net = O.OracleNet(cfg, precision)
    for t in range(gap + 5):
        if t in (0, gap):
            net.force_next([0], "replace")
        net.step(1)
    fired = any(1 in s for s in net.spikes())
    assert fired == fires


@pytest.mark.parametrize("delay", [1, 2, 3, 15])
def test_chain_latency(delay):
    """Reading R2 (step order / latency): A->B->C with suprathreshold weights; A forced at
    t0 makes B fire at t0+delay and C at t0+2 delay."""
    rules = [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0), W.Rule((1, 2), (2, 3), W.FIXED_PROB, 1.0)]
    cfg = _cfg(W.BRUNEL, 3, 3, rules, _brunel_params(JE=25.0, vlo=0.0, vhi=0.0), delay=delay)
    net = O.OracleNet(cfg)
    t0 = 5
    for t in range(t0 + 2 * delay + 3):
        if t == t0:
            net.force_next([0], "replace")
        net.step(1)
    times = {i: [t for t, s in enumerate(net.spikes()) if i in s] for i in range(3)}
    assert times == {0: [t0], 1: [t0 + delay], 2: [t0 + 2 * delay]}


def test_threshold_is_inclusive():
    """Reading R4: V >= theta spikes.  Leak disabled (tau = 1e300 -> h rounds to 0 in
    fp32) and dyadic weights: five inputs of 4 mV give V = 20 = theta exactly."""
    cfg = _cfg(W.BRUNEL, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0)],
               _brunel_params(tau=1e300, JE=4.0, vlo=0.0, vhi=0.0, tref=0.1))
    net = O.OracleNet(cfg)
    for t in range(8):
        if t < 5:
            net.force_next([0], "replace")
        net.step(1)
    t1 = [t for t, s in enumerate(net.spikes()) if 1 in s]
    assert t1 == [5]


@pytest.mark.parametrize("precision,tol", [("ref64", 1e-10), ("mirror32", 1e-5)])
def test_coba_fixed_point_closed_form(precision, tol):
    """Vogels COBA (reading R3): with frozen conductances (tau_e = tau_i = 1e300) the
    Euler map v' = v + h((E_L-v) + ge(E_e-v) + gi(E_i-v)) has the same fixed point as the
    ODE, v* = (E_L + ge E_e + gi E_i)/(1+ge+gi), approached as (1 - h(1+ge+gi))^k."""
    prm = list(W.vogels_params())
    prm[7] = prm[8] = 1e300       # tau_e, tau_i: no decay
    prm[2] = 1e9                  # V_t: never fire
    cfg = _cfg(W.VOGELS, 1, 1, [], prm)
    net = O.OracleNet(cfg, precision)
    ge, gi, v0 = 0.5, 0.25, -55.0
    net.set_state(O.F_GE, [ge]); net.set_state(O.F_GI, [gi]); net.set_state(O.F_V, [v0])
    EL, Ee, Ei = prm[1], prm[5], prm[6]
    vstar = (EL + ge * Ee + gi * Ei) / (1 + ge + gi)
    h = 0.1 / 20.0
    for k in (1, 10, 200):
        net2 = O.OracleNet(cfg, precision)
        net2.set_state(O.F_GE, [ge]); net2.set_state(O.F_GI, [gi]); net2.set_state(O.F_V, [v0])
        net2.step(k)
        ref = vstar + (v0 - vstar) * (1 - h * (1 + ge + gi)) ** k
        assert abs(net2.state(O.F_V)[0] - ref) < tol * abs(ref)


@pytest.mark.parametrize("precision,tol", [("ref64", 1e-12), ("mirror32", 1e-5)])
def test_conductance_decay_closed_form(precision, tol):
    """Vogels synaptic conductances decay as g_k = g_0 (1 - dt/tau)^k without input."""
    prm = list(W.vogels_params()); prm[2] = 1e9
    cfg = _cfg(W.VOGELS, 1, 1, [], prm)
    net = O.OracleNet(cfg, precision)
    net.set_state(O.F_GE, [3.0]); net.set_state(O.F_GI, [30.0])
    net.step(300)
    assert abs(net.state(O.F_GE)[0] - 3.0 * (1 - 0.1 / 5.0) ** 300) < tol
    assert abs(net.state(O.F_GI)[0] - 30.0 * (1 - 0.1 / 10.0) ** 300) < 30 * tol


def test_vogels_refractory_hold():
    """t_ref = 5 ms = 50 steps: after a spike v is held at V_r for 50 steps (reading R5)."""
    prm = list(W.vogels_params())
    cfg = _cfg(W.VOGELS, 1, 1, [], prm)
    net = O.OracleNet(cfg)
    net.set_state(O.F_V, [-49.0]); net.set_state(O.F_GE, [20.0])
    net.step(1)
    assert list(net.spikes()[0]) == [0]
    for _ in range(50):
        net.step(1)
        assert net.state(O.F_V)[0] == np.float32(-60.0)
    net.step(1)
    assert net.state(O.F_V)[0] > -60.0


def test_init_uniform():
    """Reading R15: initial states uniform on [lo, hi) (KS test), fields independent."""
    net = O.OracleNet(W.vogels(4000, seed=2))
    v, ge, gi = net.state(O.F_V), net.state(O.F_GE), net.state(O.F_GI)
    assert v.min() >= -60 and v.max() < -50 and ge.min() >= 0 and ge.max() < 8 and gi.max() < 40
    assert st.kstest((v + 60) / 10, "uniform").pvalue > 1e-3
    assert st.kstest(ge / 8, "uniform").pvalue > 1e-3
    assert abs(np.corrcoef(v, ge)[0, 1]) < 0.1


# --------------------------------------------------------------- delivery pins
def _adj(rp, tg, n):
    rows = np.repeat(np.arange(n), np.diff(rp.astype(np.int64)))
    return sp.csr_matrix((np.ones(len(tg), dtype=np.int64), (rows, tg.astype(np.int64))), shape=(n, n))


def test_delivery_is_spmv_packed_receptors():
    """Delivery = SpMV ("delivered to all neighbors in said row"; reading R10):
    after step t the slot read at t+delay holds A_E^T 1[S_t] + 65536 A_I^T 1[S_t], and
    the delivered-event count is sum_s rowlen(s)."""
    cfg = W.brunel(2000, 0.1, seed=7, delay=3)
    net = O.OracleNet(cfg)
    rp, tg = net.csr()
    A = _adj(rp, tg, cfg.n)
    for _ in range(40):
        net.step(1)
        s = net.spikes()[-1].astype(np.int64)
        x = np.zeros(cfg.n, dtype=np.int64)
        x[s] = 1
        xe, xi = x.copy(), x.copy()
        xe[cfg.n_exc:] = 0
        xi[:cfg.n_exc] = 0
        want = A.T @ xe + 65536 * (A.T @ xi)
        got, _ = net.input(cfg.delay - 1)
        assert np.array_equal(got.astype(np.int64), want)
        assert net.delivered()[-1] == np.diff(rp.astype(np.int64))[s].sum()


def test_synth_accumulator_is_spmv_and_activity():
    """Synth (reading R12): fired count per step ~ Binomial(N, a) within 5 sigma;
    accumulators equal A^T (sum of spike indicators over steps 0..T-1-delay)."""
    n, k, a, T = 20000, 31, 0.005, 200
    cfg = W.synth(n, k, a, seed=13)
    net = O.OracleNet(cfg)
    net.step(T)
    spikes = net.spikes()
    counts = np.array([len(s) for s in spikes])
    mu, sd = n * a, np.sqrt(n * a * (1 - a))
    assert np.all(np.abs(counts - mu) < 5 * sd + 1)
    assert abs(counts.mean() - mu) < 5 * sd / np.sqrt(T)
    x = np.zeros(n, dtype=np.int64)
    for s in spikes[:T - cfg.delay]:
        x[s] += 1
    rp, tg = net.csr()
    assert np.array_equal(net.state(O.F_ACC).astype(np.int64), _adj(rp, tg, n).T @ x)


def test_brunel_rate_gate():
    """Coarse behaviour gate: Brunel stays in (0.1, 100) Hz.
    Absolute rates are parity-unpinned (the paper prints none, R7)."""
    cfg = W.brunel(5000, 0.1, seed=3)
    net = O.OracleNet(cfg)
    net.step(2000)
    counts = np.array([len(s) for s in net.spikes()])[500:]
    rate = counts.mean() / cfg.n / 1e-4
    assert 0.1 < rate < 100


# ------------------------------------------------------------------------ STDP
def _stdp_pair_cfg(ap=0.01, am=0.0105):
    prm = _brunel_params(JE=0.0, vlo=0.0, vhi=0.0) + (20.0, 20.0, ap, am, 1.0, 0.5)
    return _cfg(W.BRUNEL_PLUS, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0, plastic=True)], prm)


@pytest.mark.parametrize("delta", [1, 5, 40])
def test_stdp_isolated_pairs(delta):
    """Pair-based STDP (reading R13): pre at t0, post at t0+delta gives
    dw = A+ a+^delta; post then pre gives dw = -A- a-^delta, with a = exp(-dt/tau)."""
    a = np.exp(-0.1 / 20.0)
    for order, sign, amp in (("pre-post", 1, 0.01), ("post-pre", -1, 0.0105)):
        net = O.OracleNet(_stdp_pair_cfg(), "ref64")
        first, second = ([0], [1]) if order == "pre-post" else ([1], [0])
        for t in range(3 + delta + 2):
            if t == 3:
                net.force_next(first, "replace")
            elif t == 3 + delta:
                net.force_next(second, "replace")
            else:
                net.force_next([], "replace")
            net.step(1)
        dw = net.weights()[0] - 0.5
        assert abs(dw - sign * amp * a ** delta) < 1e-12


def test_stdp_disabled_equals_brunel_and_weights_clamped():
    """A+ = A- = 0 reproduces the static Brunel spike train with the same rules (SPEC
    S:312); with STDP on, weights stay in [0, w_max]; the fixed-point plastic
    input equals the float sum of weights within n 2^-33 (reading R10)."""
    n = 2000
    off = W.brunel_plus(n, 0.1, seed=5, stdp_on=False)
    static = W.NetConfig("s", W.BRUNEL, n, off.n_exc,
                         tuple(W.Rule(r.src, r.dst, r.kind, r.p) for r in off.rules),
                         0.1, off.delay, off.seed, 0.0, off.params[:10])
    a, b = O.OracleNet(off), O.OracleNet(static)
    a.step(300); b.step(300)
    sa, sb = a.spikes(), b.spikes()
    assert sum(len(s) for s in sa) > 0
    assert all(np.array_equal(x, y) for x, y in zip(sa, sb))
    on = O.OracleNet(W.brunel_plus(n, 0.1, seed=5))
    on.step(300)
    w = on.weights()[on.plastic_flags() == 1]
    wmax = W.brunel_plus(n).params[14]
    assert w.min() >= 0 and w.max() <= np.float32(wmax)
    assert np.any(w != np.float32(W.brunel_plus(n).params[15]))


# ------------------------------------------------ update-rule pins (round 2)
def _vogels_params_frozen_v(**kw):
    prm = list(W.vogels_params())
    prm[2] = 1e9                               # V_t: the target never fires
    for i, v in kw.items():
        prm[i] = v
    return prm


@pytest.mark.parametrize("precision,tol", [("ref64", 1e-14), ("mirror32", 2e-6)])
def test_vogels_conductance_jump(precision, tol):
    """Vogels COBA input (readings R3/R10; P:395 defers the model to [vogels2005]): n_e
    excitatory and n_i inhibitory spikes arriving at step t raise the conductances by
    dg_e n_e and dg_i n_i before the Euler step, which then uses the raised values, and
    the conductances decay afterwards:
        ge' = ge0 + dg_e n_e,  gi' = gi0 + dg_i n_i,
        v   = v0 + h((E_L - v0) + ge'(E_e - v0) + gi'(E_i - v0)),
        ge  = ge'(1 - dt/tau_e),  gi = gi'(1 - dt/tau_i).
    n_e = 2 != n_i = 3, dg_e != dg_i and tau_e != tau_i, so swapping the two receptors
    anywhere (unpacking, weights or decay) changes the result."""
    prm = _vogels_params_frozen_v()
    # sources 0,1 excitatory; 2,3,4 inhibitory; target 5 (n_exc = 2)
    rules = [W.Rule((0, 2), (5, 6), W.FIXED_PROB, 1.0), W.Rule((2, 5), (5, 6), W.FIXED_PROB, 1.0)]
    cfg = _cfg(W.VOGELS, 6, 2, rules, prm)
    net = O.OracleNet(cfg, precision)
    net.force_next([0, 1, 2, 3, 4], "replace")
    net.step(1)                                 # step 0: the five sources fire, delivered for step 1
    ge0, gi0, v0 = 0.75, 1.5, -55.0
    for f, x in ((O.F_GE, ge0), (O.F_GI, gi0), (O.F_V, v0)):
        s = net.state(f).copy(); s[5] = x; net.set_state(f, s)
    net.step(1)
    dge, dgi, EL, Ee, Ei = prm[9], prm[10], prm[1], prm[5], prm[6]
    h, ke, ki = 0.1 / prm[0], 0.1 / prm[7], 0.1 / prm[8]
    ge1, gi1 = ge0 + dge * 2, gi0 + dgi * 3
    v = v0 + h * ((EL - v0) + ge1 * (Ee - v0) + gi1 * (Ei - v0))
    got = {f: float(net.state(f)[5]) for f in (O.F_GE, O.F_GI, O.F_V)}
    assert abs(got[O.F_GE] - ge1 * (1 - ke)) <= tol * ge1
    assert abs(got[O.F_GI] - gi1 * (1 - ki)) <= tol * gi1
    assert abs(got[O.F_V] - v) <= tol * abs(v)


def test_brunel_drive_is_poisson():
    """Brunel external drive (reading R12): per neuron and step n_ext ~ Poisson(lambda)
    by inversion of Philox words against the CDF table.  With no leak (tau = 1e300:
    h rounds to 0 in fp32), J_E = 1 (dyadic), no refractoriness and an unreachable
    threshold, each step raises V by exactly n_ext, so the V increments of 1000
    unconnected neurons over 100 steps are 1e5 Poisson draws: chi-square against the
    Poisson pmf (pooled bins with >= 5 expected) p > 1e-4, mean within 5 sigma."""
    n, T = 1000, 100
    for lam in (2.0, 16.0):
        prm = _brunel_params(tau=1e300, JE=1.0, theta=1e30, tref=0.0, lam=lam, vlo=0.0, vhi=0.0)
        net = O.OracleNet(_cfg(W.BRUNEL, n, n, [], prm, seed=17))
        prev = net.state(O.F_V).astype(np.float64)
        draws = []
        for _ in range(T):
            net.step(1)
            cur = net.state(O.F_V).astype(np.float64)
            draws.append(cur - prev)
            prev = cur
        x = np.concatenate(draws)
        assert np.all(x == np.round(x)) and x.min() >= 0
        x = x.astype(np.int64)
        m = x.size
        assert abs(x.mean() - lam) < 5 * np.sqrt(lam / m)
        kmax = int(x.max()) + 1
        obs = np.bincount(x, minlength=kmax + 1).astype(np.float64)
        pmf = st.poisson.pmf(np.arange(kmax + 1), lam)
        pmf[-1] += st.poisson.sf(kmax, lam)
        exp = pmf * m
        # pool the tails until every bin expects >= 5
        lo = 0
        while exp[:lo + 1].sum() < 5:
            lo += 1
        hi = kmax
        while exp[hi:].sum() < 5:
            hi -= 1
        o = np.concatenate(([obs[:lo + 1].sum()], obs[lo + 1:hi], [obs[hi:].sum()]))
        e = np.concatenate(([exp[:lo + 1].sum()], exp[lo + 1:hi], [exp[hi:].sum()]))
        chi2 = ((o - e) ** 2 / e).sum()
        assert st.chi2.sf(chi2, len(o) - 1) > 1e-4, (lam, chi2, len(o))


@pytest.mark.parametrize("precision", ["ref64", "mirror32"])
def test_brunel_inhibitory_weight(precision):
    """Brunel inhibitory coupling (reading R7, Brunel 2000 model A: J_I = -g J_E): with
    no leak and no drive, one excitatory and two inhibitory spikes arriving together
    change V by J_E - 2 g J_E exactly (J_E = 0.5, g = 5: 10 -> 5.5; dyadic values)."""
    prm = _brunel_params(tau=1e300, JE=0.5, g=5.0, lam=0.0, vlo=10.0, vhi=10.0, theta=1e9)
    rules = [W.Rule((0, 3), (3, 4), W.FIXED_PROB, 1.0)]
    cfg = _cfg(W.BRUNEL, 4, 1, rules, prm)      # 0 excitatory, 1 and 2 inhibitory
    net = O.OracleNet(cfg, precision)
    net.force_next([0, 1, 2], "replace")
    net.step(1)
    assert net.state(O.F_V)[3] == 10.0
    net.step(1)
    assert net.state(O.F_V)[3] == 10.0 + 0.5 - 2 * 5.0 * 0.5
    # inhibitory only: two spikes of J_I = -2.5
    net.force_next([1, 2], "replace")
    net.step(2)
    assert net.state(O.F_V)[3] == 5.5 - 5.0


@pytest.mark.parametrize("G,S", [(1, 1), (3, 32)])
def test_sampled_rows_and_columns_match_csr(G, S):
    """The full-size checkers orc_row / orc_col (reading R17) regenerate exactly the rows
    and columns of the built CSR, for fixed-probability and fixed-in-degree rules, with
    and without the ownership filter."""
    for cfg in (W.brunel(700, 0.1, seed=21), W.synth(900, 17, seed=22)):
        full_rp, full_tg = O.OracleNet(cfg).csr()
        for g in range(G):
            part = (g, G, S) if G > 1 else None
            rp, tg = O.OracleNet(cfg, part=part).csr()
            for s in range(0, cfg.n, 7):
                assert np.array_equal(O.row(cfg, s, part), tg[rp[s]:rp[s + 1]])
        src = np.repeat(np.arange(cfg.n), np.diff(full_rp.astype(np.int64)))
        order = np.lexsort((src, full_tg))
        tg_sorted, src_sorted = full_tg[order], src[order]
        starts = np.searchsorted(tg_sorted, np.arange(cfg.n + 1))
        for j in range(0, cfg.n, 11):
            assert np.array_equal(O.col(cfg, j), src_sorted[starts[j]:starts[j + 1]])


def test_synth_checkers_match_simulation():
    """The full-size synth checkers (reading R17) equal the simulated network:
    orc_synth_fired(t) is the spike set of step t and orc_synth_acc(j, T) the accumulator
    of target j after T steps, for delay 1 and delay 3."""
    for delay in (1, 3):
        cfg = W.synth(3000, 23, 0.01, seed=31, delay=delay)
        net = O.OracleNet(cfg)
        T = 60
        net.step(T)
        sp_ = net.spikes()
        for t in (0, 1, 17, T - 1):
            assert np.array_equal(O.synth_fired(cfg, t), sp_[t])
        acc = net.state(O.F_ACC)
        for j in range(0, cfg.n, 97):
            assert O.synth_acc(cfg, j, T) == int(acc[j])


# ------------------------------------------------ per-synapse delays (reading R19)
def test_per_synapse_delay_chain():
    """Reading R19 (P:485 per-synapse delays): A -> B with delay 2, B -> C with delay 5
    (rule delay ranges), the network default 1 unused: A forced at t0 fires B at t0 + 2
    and C at t0 + 7 (the single-delay chain of reading R2 generalised)."""
    rules = [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0, delay_min=2, delay_max=2),
             W.Rule((1, 2), (2, 3), W.FIXED_PROB, 1.0, delay_min=5, delay_max=5)]
    cfg = _cfg(W.BRUNEL, 3, 3, rules, _brunel_params(JE=25.0, vlo=0.0, vhi=0.0), delay=1)
    net = O.OracleNet(cfg)
    assert net.ring_slots == 6
    t0 = 4
    for t in range(t0 + 10):
        if t == t0:
            net.force_next([0], "replace")
        net.step(1)
    times = {i: [t for t, s in enumerate(net.spikes()) if i in s] for i in range(3)}
    assert times == {0: [t0], 1: [t0 + 2], 2: [t0 + 7]}


def test_per_synapse_delays_uniform_and_default():
    """Delays of a ranged rule are uniform on [dmin, dmax] (chi-square over 4e4
    synapses); a rule without a range uses the network delay."""
    n = 400
    rules = [W.Rule((0, 320), (0, n), W.FIXED_PROB, 0.3, delay_min=3, delay_max=10),
             W.Rule((320, n), (0, n), W.FIXED_PROB, 0.3)]
    cfg = _cfg(W.BRUNEL, n, 320, rules, _brunel_params(), delay=2, seed=9)
    net = O.OracleNet(cfg)
    rp, tg = net.csr()
    d = net.delays().astype(np.int64)
    src = np.repeat(np.arange(n), np.diff(rp.astype(np.int64)))
    exc, inh = d[src < 320], d[src >= 320]
    assert np.all(inh == 2) and exc.min() == 3 and exc.max() == 10
    obs = np.bincount(exc - 3, minlength=8)
    assert st.chisquare(obs).pvalue > 1e-4
    assert net.ring_slots == 11


def test_per_synapse_delivery_is_per_delay_spmv():
    """Delivery with per-synapse delays ("transmit 1-step old spikes via the first
    adjacency list, 2-steps old spikes via the second ... "): one forced spike set at step
    0 lands, for every delay d, in the slot of step d as A_d^T 1[S_0] (packed receptors),
    A_d the adjacency restricted to synapses of delay d."""
    n = 600
    rules = [W.Rule((0, 480), (0, n), W.FIXED_PROB, 0.1, delay_min=1, delay_max=6),
             W.Rule((480, n), (0, n), W.FIXED_PROB, 0.1, delay_min=2, delay_max=4)]
    cfg = _cfg(W.BRUNEL, n, 480, rules, _brunel_params(theta=1e9), delay=1, seed=12)
    net = O.OracleNet(cfg)
    rp, tg = net.csr()
    d = net.delays().astype(np.int64)
    rows = np.repeat(np.arange(n), np.diff(rp.astype(np.int64)))
    rng = np.random.default_rng(5)
    ids = np.sort(rng.choice(n, 150, replace=False))
    net.force_next(ids, "replace")
    net.step(1)
    x = np.zeros(n, dtype=np.int64)
    x[ids] = 1
    q = np.where(rows < 480, 1, 65536)
    for dd in range(1, 7):
        sel = d == dd
        A = sp.csr_matrix(((q * x[rows])[sel], (rows[sel], tg[sel].astype(np.int64))), shape=(n, n))
        want = np.asarray(A.sum(axis=0)).ravel()
        got, _ = net.input(dd - 1)
        assert np.array_equal(got.astype(np.int64), want), dd


def test_synth_checkers_with_per_synapse_delays():
    """orc_synth_acc honours per-synapse delays: equal to the simulated accumulators."""
    base = W.synth(2000, 19, 0.02, seed=41)
    cfg = W.NetConfig("sd", W.SYNTH, 2000, 2000,
                      (W.Rule((0, 2000), (0, 2000), W.FIXED_INDEGREE, k=19, delay_min=1, delay_max=5),),
                      0.1, 1, 41, 0.02, ())
    net = O.OracleNet(cfg)
    T = 40
    net.step(T)
    acc = net.state(O.F_ACC)
    for j in range(0, 2000, 83):
        assert O.synth_acc(cfg, j, T) == int(acc[j])
    assert base.n == cfg.n


# ------------------------------------------ event-driven STDP traces (reading R13)
def test_stdp_traces_closed_form():
    """Reading R13 (event-driven traces): after spikes at steps t_k the pre and post traces at
    step T are X(T) = sum_{t_k < T} exp(-(T - t_k) dt / tau+) and Y(T) likewise with tau-
    (ref64 within 1e-12; a spike at T itself is not yet counted)."""
    prm = _brunel_params(JE=0.0, vlo=0.0, vhi=0.0) + (20.0, 35.0, 0.01, 0.0105, 1.0, 0.5)
    cfg = _cfg(W.BRUNEL_PLUS, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0, plastic=True)], prm)
    net = O.OracleNet(cfg, "ref64")
    times = [3, 4, 17, 60, 61, 200]
    for t in range(260):
        net.force_next([0] if t in times else [], "replace")
        net.step(1)
        T = t + 1
        if T in (4, 18, 61, 150, 201, 260):
            past = [tk for tk in times if tk < T]
            for f, tau in ((O.F_XTR, 20.0), (O.F_YTR, 35.0)):
                want = sum(np.exp(-(T - tk) * 0.1 / tau) for tk in past)
                assert abs(net.state(f)[0] - want) < 1e-12, (T, f)
            assert net.state(O.F_XTR)[1] == 0.0


def test_stdp_cumulative_pair_sum():
    """Pair STDP over spike trains (reading R13, no clamping): the final weight is
    w0 + sum_post A+ X_pre(t_post) - sum_pre A- Y_post(t_pre), with the traces' closed
    forms, potentiation before depression at equal steps (ref64 within 1e-12)."""
    ap, am = 0.002, 0.0021
    prm = _brunel_params(JE=0.0, vlo=0.0, vhi=0.0) + (20.0, 20.0, ap, am, 10.0, 0.5)
    cfg = _cfg(W.BRUNEL_PLUS, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0, plastic=True)], prm)
    net = O.OracleNet(cfg, "ref64")
    pre, post = [5, 30, 31, 90, 140], [10, 31, 32, 100, 141, 160]
    for t in range(200):
        ids = ([0] if t in pre else []) + ([1] if t in post else [])
        net.force_next(ids, "replace")
        net.step(1)
    a = np.exp(-0.1 / 20.0)
    tr = lambda ts, T: sum(a ** (T - x) for x in ts if x < T)
    want = 0.5 + sum(ap * tr(pre, tp) for tp in post) - sum(am * tr(post, tq) for tq in pre)
    assert abs(net.weights()[0] - want) < 1e-12
