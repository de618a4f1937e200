"""The paper-fixed hand-built networks (north star: "hand-built 3-5 neuron networks with
known spike times") run through the CUDA path and compared with BOTH the closed form and
the oracle (mirror32, bit-exact), in the small-network one-CTA kernel and in the tiled
fused kernel.  The oracle-side pins of the same networks are in test_oracle_pins.py."""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu

PATHS = [dict(), dict(tile_width=32)]           # k_small (when it applies) / tiled fused kernel
PATH_IDS = ["default", "tiled"]


@pytest.fixture(scope="module")
def S():
    from paper_2102_04681_b200 import build as B
    B.build()
    from paper_2102_04681_b200 import spice
    return spice


def _cfg(model, n, n_exc, rules, params, delay=1, seed=3):
    return W.NetConfig("hand", model, n, n_exc, tuple(rules), 0.1, delay, seed, 0.0, tuple(params))


def _bp(**kw):
    p = dict(tau=20.0, VL=0.0, theta=20.0, Vr=10.0, tref=2.0, JE=0.1, g=5.0, lam=0.0, vlo=0.0, vhi=0.0)
    p.update(kw)
    return (p["tau"], p["VL"], p["theta"], p["Vr"], p["tref"], p["JE"], p["g"], p["lam"], p["vlo"], p["vhi"])


def _run_both(S, cfg, T, forcing, kw):
    """Step the GPU network and the oracle T steps with the same teacher forcing
    (forcing(t) -> (ids, mode) or None); return both spike trains."""
    o = O.OracleNet(cfg)
    with S.Network(cfg, record_steps=T, **kw) as net:
        for t in range(T):
            f = forcing(t)
            if f is not None:
                o.force_next(f[0], f[1])
                net.force_next(f[0], f[1])
            o.step(1)
            net.step(1)
        got = net.read_spikes(0, T)
        state = {"v": net.state(S.FIELD_V)}
        if cfg.model == W.VOGELS:
            state["ge"], state["gi"] = net.state(S.FIELD_GE), net.state(S.FIELD_GI)
        if cfg.model == W.BRUNEL_PLUS:
            state["w"] = net.weights()
    want = o.spikes()
    assert all(np.array_equal(a, b) for a, b in zip(got, want))
    return got, o, state


@pytest.mark.parametrize("kw", PATHS, ids=PATH_IDS)
@pytest.mark.parametrize("delay", [1, 2, 3, 15])
def test_chain_latency(S, delay, kw):
    """Reading R2: A -> B -> C (suprathreshold); A forced at t0 fires B at t0 + delay and
    C at t0 + 2 delay."""
    rules = [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0), W.Rule((1, 2), (2, 3), W.FIXED_PROB, 1.0)]
    cfg = _cfg(W.BRUNEL, 3, 3, rules, _bp(JE=25.0), delay=delay)
    t0 = 5
    got, _, _ = _run_both(S, cfg, t0 + 2 * delay + 3, lambda t: ([0], "replace") if t == t0 else None, kw)
    times = {i: [t for t, s in enumerate(got) if i in s] for i in range(3)}
    assert times == {0: [t0], 1: [t0 + delay], 2: [t0 + 2 * delay]}


@pytest.mark.parametrize("kw", PATHS, ids=PATH_IDS)
def test_threshold_is_inclusive(S, kw):
    """Reading R4 (V >= theta): no leak, five dyadic inputs of 4 mV reach theta = 20
    exactly and fire; a '>' comparison would never fire."""
    cfg = _cfg(W.BRUNEL, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0)], _bp(tau=1e300, JE=4.0, tref=0.1))
    got, _, _ = _run_both(S, cfg, 8, lambda t: ([0], "replace") if t < 5 else None, kw)
    assert [t for t, s in enumerate(got) if 1 in s] == [5]


@pytest.mark.parametrize("kw", PATHS, ids=PATH_IDS)
def test_isi_constant_drive(S, kw):
    """Reading R5: constant drive 0.15 mV/step from a source forced every step; after each
    spike the neuron is held R = 20 steps and re-crosses theta after 139 integration
    steps: ISI = 159."""
    cfg = _cfg(W.BRUNEL, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0)], _bp(JE=0.15, vlo=10.0, vhi=10.0))
    got, _, _ = _run_both(S, cfg, 700, lambda t: ([0], "add"), kw)
    t1 = [t for t, s in enumerate(got) if 1 in s]
    assert len(t1) >= 3 and np.all(np.diff(t1) == 20 + 139)


@pytest.mark.parametrize("kw", PATHS, ids=PATH_IDS)
@pytest.mark.parametrize("gap,fires", [(80, True), (81, False)])
def test_coincidence_window(S, gap, fires, kw):
    """Reading R6: two 12 mV inputs into a neuron at rest fire it iff the gap <= 80 steps."""
    cfg = _cfg(W.BRUNEL, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0)], _bp(JE=12.0))
    got, _, _ = _run_both(S, cfg, gap + 5, lambda t: ([0], "replace") if t in (0, gap) else None, kw)
    assert any(1 in s for s in got) == fires


@pytest.mark.parametrize("kw", PATHS, ids=PATH_IDS)
def test_vogels_conductance_jump(S, kw):
    """Readings R3/R10: 2 excitatory + 3 inhibitory spikes into one Vogels neuron; the
    GPU's ge, gi, v equal the oracle's bit for bit and the closed form within fp32."""
    prm = list(W.vogels_params())
    prm[2] = 1e9
    rules = [W.Rule((0, 2), (5, 6), W.FIXED_PROB, 1.0), W.Rule((2, 5), (5, 6), W.FIXED_PROB, 1.0)]
    cfg = _cfg(W.VOGELS, 6, 2, rules, prm)
    got, o, st = _run_both(S, cfg, 2, lambda t: ([0, 1, 2, 3, 4], "replace") if t == 0 else None, kw)
    for f, of in (("ge", O.F_GE), ("gi", O.F_GI), ("v", O.F_V)):
        assert np.array_equal(st[f], o.state(of)), f
    ge0, gi0 = o.state(O.F_GE), o.state(O.F_GI)
    assert ge0[5] > 0 and gi0[5] > 0


@pytest.mark.parametrize("kw", PATHS, ids=PATH_IDS)
def test_brunel_inhibitory_weight(S, kw):
    """Reading R7: one excitatory and two inhibitory spikes change V by J_E - 2 g J_E
    exactly (10 -> 5.5)."""
    prm = _bp(tau=1e300, JE=0.5, g=5.0, vlo=10.0, vhi=10.0, theta=1e9)
    cfg = _cfg(W.BRUNEL, 4, 1, [W.Rule((0, 3), (3, 4), W.FIXED_PROB, 1.0)], prm)
    got, o, st = _run_both(S, cfg, 2, lambda t: ([0, 1, 2], "replace") if t == 0 else None, kw)
    assert st["v"][3] == np.float32(5.5)


@pytest.mark.parametrize("delta", [1, 5, 40])
@pytest.mark.parametrize("order", ["pre-post", "post-pre"])
def test_stdp_isolated_pair(S, delta, order):
    """Reading R13: an isolated pair at distance delta changes the plastic
    weight by +A+ a+^delta (pre before post) or -A- a-^delta (post before pre); GPU weight
    bit-identical to the oracle's mirror32 weight, and within fp32 of the closed form."""
    prm = _bp(JE=0.0) + (20.0, 20.0, 0.01, 0.0105, 1.0, 0.5)
    cfg = _cfg(W.BRUNEL_PLUS, 2, 2, [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0, plastic=True)], prm)
    first, second = ([0], [1]) if order == "pre-post" else ([1], [0])

    def forcing(t):
        return (first if t == 3 else second if t == 3 + delta else [], "replace")
    _, o, st = _run_both(S, cfg, 3 + delta + 2, forcing, {})
    assert st["w"][0] == o.weights()[0]
    a = np.exp(-0.1 / 20.0)
    dw = 0.01 * a ** delta if order == "pre-post" else -0.0105 * a ** delta
    assert abs(float(st["w"][0]) - (0.5 + dw)) < 1e-6
