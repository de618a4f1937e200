"""Per-synapse delays (reading R19) on the GPU
against the oracle, bit-exact: delays of every synapse, spike trains, states and every
input slot of the ring, for every kernel path (fused delta_min = 1 and delta_min > 1,
cluster tiles, unfused, paper-style global atomics, Brunel+ STDP, PEER-exchange ranks)."""
import dataclasses

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2102_04681_b200 import build as B
    B.build()
    from paper_2102_04681_b200 import spice
    return spice


def _with_delays(cfg, ranges, delay=None):
    rules = tuple(dataclasses.replace(r, delay_min=lo, delay_max=hi) if (lo or hi) else r
                  for r, (lo, hi) in zip(cfg.rules, ranges))
    return dataclasses.replace(cfg, rules=rules, delay=cfg.delay if delay is None else delay)


CASES = {
    # min delay 1: the fused kernel's shared-memory path plus ring arrivals
    "brunel3000_d1to16": (_with_delays(W.brunel(3000, 0.1, seed=5), [(1, 16), (0, 0)], delay=2), {}, 300),
    # min delay 3: the ring path of the fused kernel (slot t + 3 plus longer arrivals)
    "brunel3000_d3to8": (_with_delays(W.brunel(3000, 0.1, seed=6), [(3, 8), (4, 4)]), dict(tile_width=256), 250),
    "synth20000_d1to4": (_with_delays(W.synth(20000, 31, 0.005, seed=3), [(1, 4)]), {}, 150),
    "vogels4000_d1to3": (_with_delays(W.vogels(4000), [(1, 3), (2, 2)]), {}, 300),
    "synth20000_cluster2_d1to3": (_with_delays(W.synth(20000, 31, 0.005, seed=13), [(1, 3)]),
                                  dict(tile_width=2048, ctas_per_tile=2), 100),
    "brunel3000_unfused": (_with_delays(W.brunel(3000, 0.1, seed=7), [(1, 5), (0, 0)], delay=1),
                           dict(unfused=True, tile_width=512), 200),
    "brunel3000_global_atomics": (_with_delays(W.brunel(3000, 0.1, seed=8), [(2, 6), (0, 0)], delay=3),
                                  dict(global_atomics=True), 200),
    "bplus2001_d2to5": (_with_delays(W.brunel_plus(2001, 0.15, seed=7, delay=3), [(2, 5), (0, 0), (1, 4)]),
                        dict(tile_width=128), 200),
}


@pytest.mark.parametrize("name", list(CASES))
def test_delays_free_run_bit_exact(S, name):
    cfg, kw, T = CASES[name]
    o = O.OracleNet(cfg)
    rp, tg = o.csr()
    with S.Network(cfg, record_steps=T, **kw) as net:
        offs, g = net.connectivity()
        assert np.array_equal(g, tg)
        d = net.delays()
        assert np.array_equal(d.astype(np.int64), o.delays().astype(np.int64))
        assert len(np.unique(d)) > 1
        net.step(T)
        o.step(T)
        want, got = o.spikes(), net.read_spikes(0, T)
        bad = [t for t in range(T) if not np.array_equal(got[t], want[t])]
        assert not bad, f"first mismatching step {bad[0]}"
        assert sum(len(s) for s in want) > 0
        if cfg.model == W.SYNTH:
            assert np.array_equal(net.state(S.FIELD_ACC), o.state(O.F_ACC))
        else:
            assert np.array_equal(net.state(S.FIELD_V), o.state(O.F_V))
        if cfg.model == W.BRUNEL_PLUS:
            assert np.array_equal(net.weights(), np.maximum(o.weights(), 0))
        for rel in range(o.ring_slots):
            c1, p1 = net.input(rel)
            c2, p2 = o.input(rel)
            assert np.array_equal(c1, c2), rel
            assert np.array_equal(p1, p2), rel
        assert net.stats()["delivered"] == int(o.delivered().sum())


@pytest.mark.parametrize("kw", [dict(), dict(tile_width=32)], ids=["default", "tiled"])
def test_mixed_delay_chain(S, kw):
    """Reading R19 hand-built: A -> B (delay 2) -> C (delay 5) fires B at t0 + 2, C at t0 + 7."""
    rules = [W.Rule((0, 1), (1, 2), W.FIXED_PROB, 1.0, delay_min=2, delay_max=2),
             W.Rule((1, 2), (2, 3), W.FIXED_PROB, 1.0, delay_min=5, delay_max=5)]
    prm = (20.0, 0.0, 20.0, 10.0, 2.0, 25.0, 5.0, 0.0, 0.0, 0.0)
    cfg = W.NetConfig("chain", W.BRUNEL, 3, 3, tuple(rules), 0.1, 1, 3, 0.0, prm)
    T, t0 = 15, 4
    with S.Network(cfg, record_steps=T, **kw) as net:
        for t in range(T):
            if t == t0:
                net.force_next([0], "replace")
            net.step(1)
        got = net.read_spikes(0, T)
    times = {i: [t for t, s in enumerate(got) if i in s] for i in range(3)}
    assert times == {0: [t0], 1: [t0 + 2], 2: [t0 + 7]}


@pytest.mark.parametrize("name", ["brunel3000_d1to16", "synth20000_d1to4"])
def test_delays_peer_ranks(S, name):
    """Per-synapse delays with two PEER-exchange ranks on one GPU: merged spike trains
    equal the G = 1 oracle (each rank's delay lists follow its synapse slice)."""
    cfg, kw, T = CASES[name]
    T = min(T, 150)
    G, Sw = 2, 32
    nets = [S.Network(cfg, rank=g, world_size=G, slice_width=Sw, record_steps=T,
                      exchange=S.EXCHANGE_PEER, **kw) for g in range(G)]
    try:
        hs = [n.peer_handle() for n in nets]
        for n in nets:
            n.peer_connect(hs)
        for n in nets:
            n.step(T)
        o = O.OracleNet(cfg)
        o.step(T)
        want = o.spikes()
        for n in nets:
            assert all(np.array_equal(a, b) for a, b in zip(n.read_spikes(0, T), want))
    finally:
        for n in nets:
            n.free()
