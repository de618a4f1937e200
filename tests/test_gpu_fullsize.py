"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times, on
outputs the oracle can compute one by one (R17):

* Brunel 100K (~1e9 synapses): sampled rows bit-exact against the oracle's brute-force
  row; one full-size step replayed by the oracle from the GPU's state and inputs
  (update bit-exact for all 100K neurons); the input ring after delivery equals the sum of
  the oracle's rows of that step's spiking sources (every target).
* Brunel+ 50K (250M synapses, 200M plastic): the whole network free-runs bit-exact
  against the oracle past one full flush period of the lazy STDP rows (reading R13):
  every spike, every weight, membrane potentials, traces and the input rings.
* Synth 3e9 synapses (one B200): every neuron's spike train bit-exact (the oracle
  simulates the synth drive for all 1.39M neurons); the accumulators of sampled targets
  equal the spike counts of the oracle's column (in-degree sources) of that target.
"""
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


@pytest.fixture(scope="module")
def brunel(S):
    cfg = W.brunel(100_000)
    net = S.Network(cfg, record_steps=64)
    yield cfg, net
    net.free()


def test_brunel100k_synapse_count_and_sampled_rows(S, brunel):
    cfg, net = brunel
    n = net.info()["n_synapses"]
    mean = sum((r.src[1] - r.src[0]) * (r.dst[1] - r.dst[0]) * r.p for r in cfg.rules)
    assert abs(n - mean) < 5 * np.sqrt(mean * 0.9)
    rng = np.random.default_rng(1)
    for s in list(rng.choice(cfg.n, 12, replace=False)) + [0, cfg.n_exc - 1, cfg.n_exc, cfg.n - 1]:
        offs, tg = net.connectivity(int(s), int(s) + 1)
        assert np.array_equal(tg, O.row(cfg, int(s))), s


def test_brunel100k_one_step_update_and_delivery(S, brunel):
    cfg, net = brunel
    T0 = 40
    net.step(T0 - net.stats()["steps"])
    v0, ref0 = net.state(S.FIELD_V), net.state(S.FIELD_REF)
    inp = [net.input(rel)[0] for rel in range(cfg.delay + 1)]
    net.step(1)
    sp = net.read_spikes(T0, T0 + 1)[0]
    # (1) oracle replays step T0 for all neurons from the GPU's state and inputs
    bare = dataclasses.replace(cfg, rules=())
    o = O.OracleNet(bare)
    o.set_state(O.F_V, v0)
    o.set_state(O.F_REF, ref0)
    o.set_time(T0)
    for rel in range(cfg.delay + 1):
        o.set_input(rel, inp[rel])
    o.step(1)
    assert np.array_equal(o.spikes()[T0], sp)
    assert np.array_equal(o.state(O.F_V), net.state(S.FIELD_V))
    assert np.array_equal(o.state(O.F_REF), net.state(S.FIELD_REF))
    assert len(sp) > 0
    # (2) the slot read at T0 + delay now holds exactly the deliveries of step T0:
    #     packed counts of the oracle's rows of the spiking sources (every target)
    want = inp[cfg.delay].astype(np.int64)     # earlier contents of that slot (zero)
    assert not want.any()
    for s in sp:
        q = 1 if s < cfg.n_exc else 65536
        np.add.at(want, O.row(cfg, int(s)).astype(np.int64), q)
    got = net.input(cfg.delay - 1)[0]
    assert np.array_equal(got.astype(np.int64), want)


def test_synth3b_spikes_and_sampled_accumulators(S):
    cfg = W.synth_weak(1)                      # 1,386,750 neurons, K = 2163, 3.0e9 synapses
    T = 60
    with S.Network(cfg, record_steps=T) as net:
        assert net.info()["n_synapses"] == cfg.n * cfg.rules[0].k
        net.step(T)
        got = net.read_spikes(0, T)
        acc = net.state(S.FIELD_ACC)
        st = net.stats()
    o = O.OracleNet(dataclasses.replace(cfg, rules=()))
    o.step(T)
    want = o.spikes()
    assert all(np.array_equal(a, b) for a, b in zip(got, want))
    counts = np.zeros(cfg.n, dtype=np.int64)
    for s in want[:T - cfg.delay]:
        counts[s] += 1
    rng = np.random.default_rng(3)
    for j in list(rng.choice(cfg.n, 24, replace=False)) + [0, cfg.n - 1]:
        src = O.col(cfg, int(j))
        assert len(src) == cfg.rules[0].k
        assert acc[int(j)] == counts[src.astype(np.int64)].sum(), j
    assert st["fired"] == sum(len(s) for s in want)
    # every delivered event is one (spike, synapse) pair: K per target on average
    assert abs(st["delivered"] / max(1, sum(len(s) for s in want)) - cfg.rules[0].k) < 0.02 * cfg.rules[0].k


def test_brunelplus50k_full_size_free_run(S):
    """Brunel+ at BASELINE configs[2]'s full size in bench.py's launch configuration: the
    oracle simulates the same 250M-synapse network (~40 ms per step on one host core) for
    1100 steps, past the 1024-step flush period, so every plastic row has been processed
    lazily (spike or flush) at least once; all state is compared bit-exact."""
    cfg = W.brunel_plus(50_000)
    T = 1100
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    with S.Network(cfg, record_steps=T) as net:
        assert net.info()["n_synapses"] == o.nnz
        net.step(T)
        got = net.read_spikes(0, T)
        bad = [t for t in range(T) if not np.array_equal(got[t], want[t])]
        assert not bad, f"first mismatching step {bad[0]}"
        assert sum(len(x) for x in want) > 100 * T
        w_gpu, w_orc = net.weights(), o.weights()
        moved = np.count_nonzero(w_orc[o.plastic_flags() == 1] != np.float32(cfg.params[15]))
        assert moved > 0
        assert np.array_equal(w_gpu, w_orc), np.flatnonzero(w_gpu != w_orc)[:10]
        del w_gpu, w_orc
        assert np.array_equal(net.state(S.FIELD_V), o.state(O.F_V))
        assert np.array_equal(net.state(S.FIELD_XTR), o.state(O.F_XTR))
        assert np.array_equal(net.state(S.FIELD_YTR), o.state(O.F_YTR))
        for rel in range(cfg.delay + 1):
            c1, p1 = net.input(rel)
            c2, p2 = o.input(rel)
            assert np.array_equal(c1, c2) and np.array_equal(p1, p2)
        assert net.stats()["delivered"] == int(o.delivered().sum())


def test_synth_g2_rank_slices_with_auto_cluster4_tiles(S):
    """The weak-scaling configuration at G = 2 (1,961,161 neurons, K = 3059, 3.0e9 synapses
    per rank) as two rank slices in one process, stepped through the G > 1 kernel sequence
    (exchange, bitmap->list + descriptors, fused delivery + update): the auto geometry must
    pick 4-CTA cluster tiles (abi.cu), and the union of the ranks' spikes and
    sampled accumulators must equal the oracle's (the definition: Bernoulli drive, column
    sums over the in-synapses)."""
    cfg, G, Sw, T = W.synth_weak(2), 2, 32, 30
    nets = [S.Network(cfg, rank=g, world_size=G, slice_width=Sw, external_exchange=True, record_steps=T)
            for g in range(G)]
    try:
        for n in nets:
            assert n.info()["ctas_per_tile"] == 4
        for n in nets:
            n.exchange_begin()
        for t in range(T):
            for d in nets:
                for s in nets:
                    d.exchange_put_from(s)
            for n in nets:
                n.exchange_end_fused() if t + 1 < T else n.exchange_end()
        got = [n.read_spikes(0, T) for n in nets]
        accs = [n.state(S.FIELD_ACC) for n in nets]
    finally:
        for n in nets:
            n.free()
    o = O.OracleNet(dataclasses.replace(cfg, rules=()))
    o.step(T)
    want = o.spikes()
    for g in range(G):
        assert all(np.array_equal(a, b) for a, b in zip(got[g], want)), g
    counts = np.zeros(cfg.n, dtype=np.int64)
    for s in want[:T - cfg.delay]:
        counts[s] += 1
    rng = np.random.default_rng(5)
    for g in range(G):
        for i in list(rng.choice(len(accs[g]), 12, replace=False)) + [0, len(accs[g]) - 1]:
            j = S.partition_local_to_global(int(i), g, G, Sw)
            src = O.col(cfg, int(j))
            assert accs[g][int(i)] == counts[src.astype(np.int64)].sum(), (g, i, j)
