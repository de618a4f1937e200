"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element on the same seeded inputs.  Static models (Vogels, Brunel, Synth) accumulate
integer receptor counts (reading R10) and update in fp32 with the paper's Euler order
(reading R3), so connectivity, spike lists, inputs and states are compared BIT-EXACT
against oracle mirror32.  Sizes span many tiles plus a ragged tail."""
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


CASES = {
    "vogels4000": (W.vogels(4000), {}, 1000),
    "vogels4000_t32_c3": (W.vogels(4000), dict(tile_width=32, ctas_per_tile=3), 400),
    "brunel3000_d15": (W.brunel(3000, 0.1, seed=5, delay=15), {}, 400),
    "brunel1001_ragged": (W.brunel(1001, 0.2, seed=2, delay=3), dict(tile_width=64), 300),
    # delay 1 Brunel: the small-network one-CTA kernel with the Poisson drive
    "brunel2000_d1_small": (W.brunel(2000, 0.1, seed=18, delay=1), {}, 300),
    "synth20000": (W.synth(20000, 31, 0.005, seed=3), {}, 200),
    "synth5003_ragged_c2": (W.synth(5003, 100, 0.02, seed=4), dict(tile_width=96, ctas_per_tile=2), 150),
    # tile wider than byte-offset entries allow: padded layout with counter-index entries
    "synth40000_wide_tile": (W.synth(40000, 31, 0.005, seed=11), dict(tile_width=16384), 60),
    # thread-block-cluster tiles (C CTAs per tile, DSMEM reduction of the tile counters)
    "synth40000_cluster2_word": (W.synth(40000, 31, 0.005, seed=12), dict(tile_width=20480, ctas_per_tile=2), 60),
    "synth20000_cluster4": (W.synth(20000, 31, 0.005, seed=13), dict(ctas_per_tile=4), 100),
    "brunel3000_d15_cluster4": (W.brunel(3000, 0.1, seed=14, delay=15), dict(tile_width=256, ctas_per_tile=4), 300),
    "vogels4000_cluster8": (W.vogels(4000, seed=15), dict(tile_width=512, ctas_per_tile=8), 300),
    "vogels_global_atomics": (W.vogels(4000, seed=9), dict(global_atomics=True), 300),
    "synth_global_atomics": (W.synth(20000, 31, 0.005, seed=8), dict(global_atomics=True), 100),
    # long enough that per-step list counters must be recycled (regression: they were not)
    "synth_global_atomics_long": (W.synth(5003, 31, 0.05, seed=16), dict(global_atomics=True), 800),
    "synth_long_unfused_c2": (W.synth(5003, 31, 0.05, seed=17), dict(unfused=True, ctas_per_tile=2), 800),
}

_oracle_cache = {}


def oracle_run(name):
    if name not in _oracle_cache:
        cfg, _, T = CASES[name]
        o = O.OracleNet(cfg)
        init = {f: o.state(f) for f in (O.F_V, O.F_GE, O.F_GI)}
        o.step(T)
        _oracle_cache[name] = (o, init)
    return _oracle_cache[name]


def assert_same_csr(net, o, rows=None):
    rp, tg = o.csr()
    offs, g = net.connectivity()
    assert np.array_equal(offs.astype(np.int64), rp.astype(np.int64) - int(rp[0]))
    assert np.array_equal(g, tg)


@pytest.mark.parametrize("name", list(CASES))
def test_connectivity_bit_exact(S, name):
    cfg, kw, _ = CASES[name]
    o = O.OracleNet(cfg)
    with S.Network(cfg, **kw) as net:
        assert net.info()["n_synapses"] == o.nnz
        assert_same_csr(net, o)


@pytest.mark.parametrize("name", [n for n in CASES if not n.startswith("synth")])
def test_initial_state_bit_exact(S, name):
    cfg, kw, _ = CASES[name]
    o = O.OracleNet(cfg)
    with S.Network(cfg, **kw) as net:
        assert np.array_equal(net.state(S.FIELD_V), o.state(O.F_V))
        if cfg.model == W.VOGELS:
            assert np.array_equal(net.state(S.FIELD_GE), o.state(O.F_GE))
            assert np.array_equal(net.state(S.FIELD_GI), o.state(O.F_GI))


@pytest.mark.parametrize("name", list(CASES))
def test_free_run_bit_exact(S, name):
    """Spike lists of every step, final state and event counters, bit-exact."""
    cfg, kw, T = CASES[name]
    o, _ = oracle_run(name)
    want = o.spikes()
    with S.Network(cfg, record_steps=T, **kw) as net:
        net.step(T)
        got = net.read_spikes(0, T)
        bad = [t for t in range(T) if not np.array_equal(got[t], want[t])]
        assert not bad, f"first mismatching step {bad[0]}: gpu {got[bad[0]][:10]} oracle {want[bad[0]][:10]}"
        st = net.stats()
        assert st["fired"] == sum(len(s) for s in want)
        assert st["delivered"] == int(o.delivered().sum())
        if cfg.model == W.SYNTH:
            assert np.array_equal(net.state(S.FIELD_ACC), o.state(O.F_ACC))
        else:
            assert np.array_equal(net.state(S.FIELD_V), o.state(O.F_V))
            assert np.array_equal(net.state(S.FIELD_REF), o.state(O.F_REF))
        if cfg.model == W.VOGELS:
            assert np.array_equal(net.state(S.FIELD_GE), o.state(O.F_GE))
            assert np.array_equal(net.state(S.FIELD_GI), o.state(O.F_GI))
        for rel in range(cfg.delay + 1):
            assert np.array_equal(net.input(rel)[0], o.input(rel)[0])
    assert sum(len(s) for s in want) > 0


@pytest.mark.parametrize("name", ["brunel3000_d15", "vogels4000", "synth20000"])
def test_teacher_forced_inputs_every_step(S, name):
    """Teacher forcing (north star: per-step synaptic input under identical spikes):
    a random spike set is forced on both sides every step; all input slots equal."""
    cfg, kw, _ = CASES[name]
    rng = np.random.default_rng(7)
    o = O.OracleNet(cfg)
    with S.Network(cfg, **kw) as net:
        for t in range(25):
            ids = np.sort(rng.choice(cfg.n, size=rng.integers(0, cfg.n // 3), replace=False)).astype(np.uint32)
            mode = "replace" if t % 2 == 0 else "add"
            o.force_next(ids, mode)
            net.force_next(ids, mode)
            o.step(1)
            net.step(1)
            assert np.array_equal(net.read_spikes(t, t + 1)[0], o.spikes()[t])
            for rel in range(cfg.delay + 1):
                assert np.array_equal(net.input(rel)[0], o.input(rel)[0]), (t, rel)


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("name", ["vogels4000", "brunel3000_d15", "synth20000", "synth20000_cluster4",
                                  "brunel3000_d15_cluster4"])
def test_virtual_ranks_match_single_gpu(S, G, name, fused):
    """G network slices on one GPU with the bitmap exchange done through the C ABI:
    slice connectivity = descriptor split, merged spike trains identical to
    the G=1 oracle (partition invariance), owned states identical."""
    cfg, kw, T = CASES[name]
    T = min(T, 200)
    o, _ = oracle_run(name)
    Sw = 32
    nets = [S.Network(cfg, rank=g, world_size=G, slice_width=Sw, external_exchange=True,
                      record_steps=T, **kw) for g in range(G)]
    try:
        for g, net in enumerate(nets):
            assert_same_csr(net, O.OracleNet(cfg, part=(g, G, Sw)))
        if fused:       # the NCCL graph's sequence: begin; (exchange, end_fused) x (T-1); exchange, end
            for n in nets:
                n.exchange_begin()
            for t in range(T):
                for d in nets:
                    for s in nets:
                        d.exchange_put_from(s)
                for n in nets:
                    n.exchange_end_fused() if t + 1 < T else n.exchange_end()
        else:
            for _ in range(T):
                for n in nets:
                    n.exchange_begin()
                for d in nets:
                    for s in nets:
                        d.exchange_put_from(s)
                for n in nets:
                    n.exchange_end()
        want = o.spikes()[:T]
        for n in nets:
            got = n.read_spikes(0, T)
            assert all(np.array_equal(a, b) for a, b in zip(got, want))
        # owned state == oracle state at the owned global IDs (oracle ran longer: rerun)
        o2 = O.OracleNet(cfg)
        o2.step(T)
        field, ofield = (S.FIELD_ACC, O.F_ACC) if cfg.model == W.SYNTH else (S.FIELD_V, O.F_V)
        full = o2.state(ofield)
        for g, n in enumerate(nets):
            ids = np.array([S.partition_local_to_global(i, g, G, Sw) for i in range(n.n_owned)])
            assert np.array_equal(n.state(field), full[ids])
        fired = sum(n.stats()["fired"] for n in nets)
        assert fired == sum(len(s) for s in want)
        delivered = sum(n.stats()["delivered"] for n in nets)
        assert delivered == int(o2.delivered().sum())
    finally:
        for n in nets:
            n.free()


def test_edge_cases(S):
    # no synapses at all; tiny N below one warp; silent synth
    base = W.brunel(20, 0.1, seed=1, delay=2)
    cfg = dataclasses.replace(base, rules=tuple(dataclasses.replace(r, p=0.0) for r in base.rules))
    o = O.OracleNet(cfg)
    with S.Network(cfg) as net:
        assert net.info()["n_synapses"] == 0
        net.step(50)
        o.step(50)
        assert all(np.array_equal(a, b) for a, b in zip(net.read_spikes(0, 50), o.spikes()))
    with S.Network(W.synth(1000, 10, 0.0, seed=1)) as net:
        net.step(40)
        assert sum(len(s) for s in net.read_spikes(0, 40)) == 0
    # record ring bounds
    with S.Network(W.synth(2000, 5, 0.01), record_steps=8) as net:
        net.step(20)
        with pytest.raises(S.SpiceError) as e:
            net.read_spikes(5, 20)
        assert e.value.status == S.ERANGE
        assert len(net.read_spikes(12, 20)) == 8
        with pytest.raises(S.SpiceError) as e:
            net.read_spikes(19, 21)
        assert e.value.status == S.ERANGE


def test_graph_chunks_equal_single_steps(S):
    """spice_step(n) replays a 32-step graph plus single steps; any split gives the same."""
    cfg = W.brunel(2000, 0.1, seed=11, delay=2)
    with S.Network(cfg, record_steps=100) as a, S.Network(cfg, record_steps=100) as b:
        a.step(100)
        for n in (1, 31, 33, 2, 32, 1):
            b.step(n)
        assert all(np.array_equal(x, y) for x, y in zip(a.read_spikes(0, 100), b.read_spikes(0, 100)))


@pytest.mark.parametrize("name", ["vogels4000", "brunel3000_d15", "synth20000"])
def test_profile_modes_keep_the_simulation_exact(S, name):
    """spice_profile advances the network through unfused, individually launched fused and
    graph-captured fused launches; every step must still equal the oracle's."""
    cfg, kw, T = CASES[name]
    o, _ = oracle_run(name)
    want = o.spikes()
    with S.Network(cfg, record_steps=T, **kw) as net:
        net.step(5)
        prof = net.profile(8)            # 8 unfused, 9 fused, 65 graph-fused steps
        assert prof["update"] > 0 and prof["deliver"] > 0
        assert prof["fused"] > 0 and prof["fused_in_graph"] > 0
        done = net.stats()["steps"]
        assert done < T
        net.step(T - done)
        got = net.read_spikes(0, T)
    bad = [t for t in range(T) if not np.array_equal(got[t], want[t])]
    assert not bad, f"first mismatching steps {bad[:5]}"
