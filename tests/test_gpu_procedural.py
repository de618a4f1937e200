"""Procedural connectivity ("only store the parameters used to
create the network and then generate adjacency data on the fly" [Knight2021]): the library
stores no rows and regenerates every spike's row segment per tile from the FIXED_PROB Philox
predicate (reading R9).  The network is the same one the stored path and the oracle build,
so everything is compared BIT-EXACT with the oracle: connectivity, delays, spike trains,
states, every input slot, delivered-event counts; single GPU and two PEER-exchange ranks."""
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


def _delays(cfg, ranges):
    return dataclasses.replace(cfg, rules=tuple(dataclasses.replace(r, delay_min=lo, delay_max=hi)
                                               for r, (lo, hi) in zip(cfg.rules, ranges)))


CASES = {
    "vogels4000": (W.vogels(4000), {}, 300),
    "brunel3000_d15": (W.brunel(3000, 0.1, seed=5, delay=15), dict(tile_width=256), 300),
    "brunel2001_ragged_d1": (W.brunel(2001, 0.15, seed=6, delay=1), dict(tile_width=96), 200),
    "brunel3000_delays": (_delays(W.brunel(3000, 0.1, seed=7), [(1, 12), (2, 3)]), {}, 250),
}


@pytest.mark.parametrize("name", list(CASES))
def test_procedural_bit_exact(S, name):
    cfg, kw, T = CASES[name]
    o = O.OracleNet(cfg)
    rp, tg = o.csr()
    with S.Network(cfg, record_steps=T, procedural=True, **kw) as net:
        assert net.info()["n_synapses"] == o.nnz
        assert net.info()["device_bytes"] < 16 * cfg.n * 64       # O(neurons): no synapse storage
        offs, g = net.connectivity(0, min(cfg.n, 300))
        assert np.array_equal(g, tg[: int(rp[min(cfg.n, 300)])])
        d = net.delays(0, min(cfg.n, 300))
        assert np.array_equal(d.astype(np.int64), o.delays()[: len(d)].astype(np.int64))
        net.step(T)
        o.step(T)
        want, got = o.spikes(), net.read_spikes(0, T)
        bad = [t for t in range(T) if not np.array_equal(got[t], want[t])]
        assert not bad, f"first mismatching step {bad[0]}"
        assert sum(len(s) for s in want) > 0
        assert np.array_equal(net.state(S.FIELD_V), o.state(O.F_V))
        for rel in range(o.ring_slots):
            assert np.array_equal(net.input(rel)[0], o.input(rel)[0]), rel
        assert net.stats()["delivered"] == int(o.delivered().sum())


def test_procedural_peer_ranks(S):
    cfg, kw, T = CASES["brunel3000_d15"]
    G, Sw = 2, 32
    nets = [S.Network(cfg, rank=g, world_size=G, slice_width=Sw, record_steps=T, procedural=True,
                      exchange=S.EXCHANGE_PEER, **kw) for g in range(G)]
    try:
        hs = [n.peer_handle() for n in nets]
        for n in nets:
            n.peer_connect(hs)
        for n in nets:
            n.step(T)
        o = O.OracleNet(cfg)
        o.step(T)
        for n in nets:
            assert all(np.array_equal(a, b) for a, b in zip(n.read_spikes(0, T), o.spikes()))
        assert sum(n.stats()["delivered"] for n in nets) == int(o.delivered().sum())
    finally:
        for n in nets:
            n.free()


def test_procedural_rejects_what_it_cannot_regenerate(S):
    with pytest.raises(S.SpiceError):
        S.Network(W.synth(2000, 10), procedural=True)             # fixed in-degree rule
    with pytest.raises(S.SpiceError):
        S.Network(W.brunel_plus(2000), procedural=True)           # STDP needs stored weights
