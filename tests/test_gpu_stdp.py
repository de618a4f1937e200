"""Brunel+ (STDP) on the GPU against the oracle's eager rule (reading
R13): pair-STDP weights, traces, plastic fixed-point inputs and spike trains BIT-EXACT
(every weight change is a single fp32 operation per synapse in a fixed order; plastic
input is int64 fixed point, reading R10)."""
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


def _stronger_stdp(cfg, scale=20.0):
    """Same network with A+/A- scaled up so that weights visibly move in a short run."""
    import dataclasses
    p = list(cfg.params)
    p[12] *= scale
    p[13] *= scale
    return dataclasses.replace(cfg, params=tuple(p))


CASES = {
    "bplus3000": (W.brunel_plus(3000, 0.1, seed=5), {}, 300),
    "bplus3000_strong_t64": (_stronger_stdp(W.brunel_plus(3000, 0.1, seed=6)), dict(tile_width=64), 300),
    "bplus2001_ragged": (_stronger_stdp(W.brunel_plus(2001, 0.15, seed=7, delay=3)), dict(tile_width=96), 200),
    # the Brunel+ 50K bench geometry's segment length (~35 entries per (row, tile))
    "bplus3000_t384": (_stronger_stdp(W.brunel_plus(3000, 0.1, seed=8)), dict(tile_width=384), 250),
    "bplus2001_t32": (_stronger_stdp(W.brunel_plus(2001, 0.15, seed=11, delay=2)), dict(tile_width=32), 200),
}


@pytest.mark.parametrize("name", list(CASES))
def test_brunel_plus_free_run_bit_exact(S, name):
    cfg, kw, T = CASES[name]
    o = O.OracleNet(cfg)
    rp, tg = o.csr()
    with S.Network(cfg, record_steps=T, **kw) as net:
        offs, g = net.connectivity()
        assert np.array_equal(g, tg)
        assert np.array_equal(net.weights(), o.weights())          # w0 on plastic, 0 elsewhere
        net.step(T)
        o.step(T)
        want = o.spikes()
        got = net.read_spikes(0, T)
        bad = [t for t in range(T) if not np.array_equal(got[t], want[t])]
        assert not bad, f"first mismatching step {bad[0]}"
        w_gpu, w_orc = net.weights(), o.weights()
        assert np.array_equal(w_gpu, w_orc), np.flatnonzero(w_gpu != w_orc)[:10]
        assert np.any(w_orc[o.plastic_flags() == 1] != np.float32(cfg.params[15]))  # STDP acted
        assert np.array_equal(net.state(S.FIELD_V), o.state(O.F_V))
        assert np.array_equal(net.state(S.FIELD_YTR), o.state(O.F_YTR))
        assert np.array_equal(net.state(S.FIELD_XTR), o.state(O.F_XTR))
        for rel in range(cfg.delay + 1):
            c1, p1 = net.input(rel)
            c2, p2 = o.input(rel)
            assert np.array_equal(c1, c2) and np.array_equal(p1, p2)
        assert net.stats()["delivered"] == int(o.delivered().sum())


@pytest.mark.parametrize("G", [2, 3])
def test_brunel_plus_virtual_ranks(S, G):
    cfg, _, T = CASES["bplus3000_strong_t64"]
    T = 150
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    Sw = 32
    nets = [S.Network(cfg, rank=g, world_size=G, slice_width=Sw, external_exchange=True,
                      record_steps=T) for g in range(G)]
    try:
        for _ in range(T):
            for n in nets:
                n.exchange_begin()
            for d in nets:
                for s in nets:
                    d.exchange_put_from(s)
            for n in nets:
                n.exchange_end()
        for n in nets:
            assert all(np.array_equal(a, b) for a, b in zip(n.read_spikes(0, T), want))
        # per-rank weights equal the oracle's weights of that rank's synapses
        for g, n in enumerate(nets):
            part = O.OracleNet(cfg, part=(g, G, Sw))
            rp, tg = part.csr()
            offs, gt = n.connectivity()
            assert np.array_equal(gt, tg)
        # weights: compare per synapse through (source, target) keys
        full_rp, full_tg = o.csr()
        wfull = o.weights()
        key = {}
        for s_ in range(cfg.n):
            for e in range(int(full_rp[s_]), int(full_rp[s_ + 1])):
                key[(s_, int(full_tg[e]))] = wfull[e]
        for g, n in enumerate(nets):
            offs, gt = n.connectivity()
            wg = n.weights()
            for s_ in range(0, cfg.n, 7):
                for e in range(int(offs[s_]), int(offs[s_ + 1])):
                    assert wg[e] == key[(s_, int(gt[e]))]
    finally:
        for n in nets:
            n.free()


def test_brunel_plus_teacher_forced_bursts(S):
    """Steps with more spikes than one staging pass of the flattened delivery holds (2048
    segments per tile per pass): forced bursts of 2500 spikes, weights, inputs and spike
    trains still bit-exact against the oracle."""
    cfg = _stronger_stdp(W.brunel_plus(3000, 0.1, seed=12))
    rng = np.random.default_rng(3)
    o = O.OracleNet(cfg)
    with S.Network(cfg, record_steps=64, tile_width=384) as net:
        for t in range(40):
            if t % 7 == 3:
                ids = np.sort(rng.choice(cfg.n, 2500, replace=False)).astype(np.uint32)
                o.force_next(ids, "add")
                net.force_next(ids, "add")
            o.step(1)
            net.step(1)
        want = o.spikes()
        got = net.read_spikes(0, 40)
        assert all(np.array_equal(x, y) for x, y in zip(got, want))
        assert max(len(x) for x in want) >= 2500
        assert np.array_equal(net.weights(), np.maximum(o.weights(), 0))
        for rel in range(cfg.delay + 1):
            c1, p1 = net.input(rel)
            c2, p2 = o.input(rel)
            assert np.array_equal(c1, c2) and np.array_equal(p1, p2)


def test_brunel_plus_persistent_kernel_matches_per_step_kernels(S):
    """The persistent Brunel+ kernel (k_plastic_run: one launch per graph replay, the update
    warps arrive at the grid barrier once t + 1 is published, spike lists and pre state in
    copies t mod 3) against one k_fused<3> per step (SPICE_NO_PERSIST=1, read when a network
    is created): spikes, weights, traces, inputs bit-identical, over replays of 1 .. 256 steps
    (300 = 256 + 32 + 8 + 4)."""
    import os
    cfg, kw, T = _stronger_stdp(W.brunel_plus(3000, 0.1, seed=21)), dict(tile_width=128), 300
    out = {}
    for persist in (True, False):
        if not persist:
            os.environ["SPICE_NO_PERSIST"] = "1"
        try:
            with S.Network(cfg, record_steps=T, **kw) as net:
                assert (net.launches(32) == 4) == persist          # one persistent launch per replay
                net.step(T)
                out[persist] = (net.read_spikes(0, T), net.weights(), net.state(S.FIELD_V),
                                net.state(S.FIELD_XTR), net.state(S.FIELD_YTR), net.input(0), net.stats())
        finally:
            os.environ.pop("SPICE_NO_PERSIST", None)
    a, b = out[True], out[False]
    assert all(np.array_equal(a[0][t], b[0][t]) for t in range(T))
    for x, y in zip(a[1:5], b[1:5]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[5][0], b[5][0]) and np.array_equal(a[5][1], b[5][1])
    assert a[6]["delivered"] == b[6]["delivered"] and a[6]["fired"] == b[6]["fired"]
    o = O.OracleNet(cfg)
    o.step(T)
    assert np.array_equal(a[1], o.weights())
    assert all(np.array_equal(a[0][t], s) for t, s in enumerate(o.spikes()))
