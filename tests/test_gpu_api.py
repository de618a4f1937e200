"""GPU tests of the C-ABI surface around the step loop: setup timing, launch accounting,
record-ring bounds and the zero-allocation read path used by bench.py's e2e leg.  The
spike trains themselves are checked against the oracle in test_gpu_parity.py."""
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


def test_setup_times_are_reported(S):
    with S.Network(W.synth(20000, 31, 0.005, seed=3)) as net:
        t = net.setup_times()
        assert 0.0 < t["gen_ms"] <= t["create_ms"]


def _decompose(n, top=256):
    """spice_step's graph decomposition: the largest power of two <= min(n, 256) first."""
    out = []
    while n:
        m = top
        while m > n:
            m //= 2
        out.append(m)
        n -= m
    return out


@pytest.mark.parametrize("kw, per_graph", [
    ({}, lambda m: 2),                                  # small network: one k_small + k_advance per replay
    (dict(tile_width=1024), lambda m: m + 2),           # tiled: update, m-1 fused, deliver, advance
    (dict(tile_width=1024, unfused=True), lambda m: 2 * m + 1),   # update + deliver per step, advance
])
def test_launch_accounting(S, kw, per_graph):
    """Every spice_step(n) runs graphs of 2^k fused steps, so a 20-step call is 16 + 4 and
    costs n + O(log n) launches, not 3 per leftover step.  With the
    persistent synth kernel (G = 1, delay 1, whole grid co-resident) a replay of m > 1
    steps is four launches: update, ONE persistent launch of m - 1 steps, deliver, advance."""
    with S.Network(W.synth(20000, 31, 0.005, seed=3), **kw) as net:
        if kw.get("tile_width") and not kw.get("unfused") and net.launches(32) == 4:
            per_graph = lambda m: 4 if m > 1 else 3      # noqa: E731 (persistent form)
        for n in (1, 20, 32, 33, 64, 300, 1000):
            assert net.launches(n) == sum(per_graph(m) for m in _decompose(n)), n
        if "unfused" not in kw:
            assert net.launches(20) <= 20 + 4


def test_prefetch_collect_double_buffer_matches_oracle(S):
    """spice_spikes_prefetch / _collect: chunked, double-buffered read-out (bench e2e leg)
    returns the same per-step lists as the oracle, including a ring wrap."""
    cfg, T, K = W.synth(5003, 31, 0.05, seed=21), 96, 12
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    ids = np.zeros(cfg.n * K, dtype=np.uint32)
    offs = np.zeros(K + 1, dtype=np.uint64)
    got = []
    with S.Network(cfg, record_steps=20, tile_width=1024) as net:
        for c in range(T // K):
            net.step(K)
            net.spikes_prefetch(c * K, (c + 1) * K, c & 1)
            if c:
                n = net.spikes_collect_into((c - 1) & 1, ids, offs)
                got += [ids[int(offs[q]):int(offs[q + 1])].copy() for q in range(K)]
                assert int(offs[K]) == n
        net.spikes_collect_into((T // K - 1) & 1, ids, offs)
        got += [ids[int(offs[q]):int(offs[q + 1])].copy() for q in range(K)]
        with pytest.raises(S.SpiceError):
            net.spikes_collect_into(0, ids, offs)              # nothing prefetched
        with pytest.raises(S.SpiceError):
            net.spikes_prefetch(0, 10, 0)                      # older than the ring
    assert all(np.array_equal(g, w) for g, w in zip(got, want))


def test_user_stream_and_torch_allocator(S):
    """spice_config.stream + SPICE_FLAG_USER_STREAM and dev_alloc/dev_free: the library
    enqueues on torch's stream and holds its buffers in torch's caching allocator; results
    are unchanged (checked against the oracle)."""
    import torch
    cfg, T = W.synth(20000, 31, 0.005, seed=3), 70
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    held = {}

    def alloc(nbytes):
        p = torch.cuda.caching_allocator_alloc(nbytes)
        held[p] = nbytes
        return p

    def free(p):
        held.pop(p)
        torch.cuda.caching_allocator_delete(p)

    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    before = torch.cuda.memory_allocated()
    with S.Network(cfg, record_steps=T, tile_width=1024, stream=s.cuda_stream, allocator=(alloc, free)) as net:
        assert net.stream == s.cuda_stream
        assert torch.cuda.memory_allocated() - before >= net.info()["device_bytes"] > 0
        net.step(T)
        got = net.read_spikes(0, T)
    assert not held and torch.cuda.memory_allocated() == before
    assert all(np.array_equal(g, w) for g, w in zip(got, want))
    # the legacy default stream works too (graphs are captured on a private stream)
    with S.Network(cfg, record_steps=T, tile_width=1024, stream=0) as net:
        net.step(T)
        got = net.read_spikes(0, T)
    assert all(np.array_equal(g, w) for g, w in zip(got, want))


def test_write_state_round_trip(S):
    """spice_write_state mirrors spice_read_state for every writable field, at an even and
    an odd step; the STDP traces are event-driven state (reading R13) and reject writes
    (the old trace write was wrong at odd steps)."""
    cfg = W.brunel_plus(2001, 0.1, seed=5)
    with S.Network(cfg, world_size=2, rank=1, external_exchange=True, tile_width=256) as net:
        rng = np.random.default_rng(0)
        for t in range(2):                      # t_host = 0, then 1 (the other trace buffer)
            if t:
                net.exchange_begin()            # one step; rank 0's bitmap stays all-zero
                net.exchange_end()
            x = rng.random(net.n_owned).astype(np.float32)
            net.write_state(S.FIELD_V, x)
            assert np.array_equal(net.state(S.FIELD_V), x), t
            for f in (S.FIELD_XTR, S.FIELD_YTR):          # event-driven traces: read-only
                net.state(f)
                with pytest.raises(S.SpiceError):
                    net.write_state(f, x)
            r = rng.integers(0, 5, net.n_owned).astype(np.uint32)
            net.write_state(S.FIELD_REF, r)
            assert np.array_equal(net.state(S.FIELD_REF), r)


def test_record_ring_bounds(S):
    cfg = W.vogels(4000)
    with S.Network(cfg, record_steps=16) as net:
        net.step(40)
        assert len(net.read_spikes(24, 40)) == 16          # the last record_steps steps
        with pytest.raises(S.SpiceError):
            net.read_spikes(20, 40)                         # older than the ring
        with pytest.raises(S.SpiceError):
            net.read_spikes(30, 41)                         # not simulated yet


def test_read_spikes_into_matches_oracle(S):
    """The e2e read path (pinned staging, reused decode buffers) step by step."""
    cfg, T = W.synth(5003, 31, 0.05, seed=21), 64
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    ids = np.zeros(cfg.n, dtype=np.uint32)
    offs = np.zeros(2, dtype=np.uint64)
    with S.Network(cfg, record_steps=8) as net:
        for t in range(T):
            net.step(1)
            k = net.read_spikes_into(t, t + 1, ids, offs)
            assert np.array_equal(ids[:k], want[t]), t


def test_prefetch_collect_beyond_the_guess(S):
    """Device-compacted read-out (chunks of >= 2^16 bitmap words): a chunk with far more
    spikes than the slot's previous chunk (forced bursts) makes collect fetch the IDs past the
    speculative copy; ETRUNC keeps the slot for a larger buffer."""
    cfg, K = W.synth(200_000, 31, 0.002, seed=4), 12
    rng = np.random.default_rng(5)
    o = O.OracleNet(cfg)
    ids = np.zeros(cfg.n * K, dtype=np.uint32)
    offs = np.zeros(K + 1, dtype=np.uint64)
    with S.Network(cfg, record_steps=32, tile_width=1024) as net:
        for c in range(4):
            for q in range(K):
                if c == 2 and q % 2 == 0:
                    f = np.sort(rng.choice(cfg.n, 150_000, replace=False)).astype(np.uint32)
                    o.force_next(f, "add")
                    net.force_next(f, "add")
                o.step(1)
                net.step(1)
            net.spikes_prefetch(c * K, (c + 1) * K, c & 1)
            if c == 2:
                small = np.zeros(10, dtype=np.uint32)
                with pytest.raises(S.SpiceError):
                    net.spikes_collect_into(c & 1, small, offs)
            n = net.spikes_collect_into(c & 1, ids, offs)
            want = o.spikes()[c * K:(c + 1) * K]
            assert n == sum(len(w) for w in want)
            for q in range(K):
                assert np.array_equal(ids[int(offs[q]):int(offs[q + 1])], want[q]), (c, q)
        assert max(len(x) for x in o.spikes()) >= 150_000


def test_compacted_readout_guards_its_ring_slots(S):
    """The compacted read-out runs on its own stream; with a ring barely larger than a chunk
    the next chunk's steps overwrite its slots and must wait for it (spice_step's guard)."""
    cfg, T, K = W.synth(200_000, 31, 0.002, seed=6), 48, 12
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    ids = np.zeros(cfg.n * K, dtype=np.uint32)
    offs = np.zeros(K + 1, dtype=np.uint64)
    got = []
    with S.Network(cfg, record_steps=16, tile_width=4096) as net:
        for c in range(T // K):
            net.step(K)
            net.spikes_prefetch(c * K, (c + 1) * K, c & 1)
            if c:
                net.spikes_collect_into((c - 1) & 1, ids, offs)
                got += [ids[int(offs[q]):int(offs[q + 1])].copy() for q in range(K)]
        net.spikes_collect_into((T // K - 1) & 1, ids, offs)
        got += [ids[int(offs[q]):int(offs[q + 1])].copy() for q in range(K)]
    assert all(np.array_equal(g, w) for g, w in zip(got, want))


@pytest.mark.parametrize("kw", [dict(tile_width=4096), dict(tile_width=20480, ctas_per_tile=2)])
def test_persistent_synth_kernel_matches_per_step_kernels_and_oracle(S, kw):
    """The persistent synth kernel (k_synth_run: one launch per graph replay, in-kernel grid
    barrier, tile counters folded into acc once per launch) against one fused kernel per step
    (SPICE_NO_PERSIST=1, read when a network is created) and the oracle: spike lists, the
    accumulators and the delivered/fired counts, over replays of 1 .. 256 steps."""
    import os
    cfg, T = W.synth(40000, 31, 0.005, seed=12), 300        # 256 + 32 + 8 + 4: every replay size
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    out = {}
    for persist in (True, False):
        if not persist:
            os.environ["SPICE_NO_PERSIST"] = "1"
        try:
            with S.Network(cfg, record_steps=T, **kw) as net:
                assert (net.launches(32) == 4) == persist          # one persistent launch per replay
                net.step(T)
                out[persist] = (net.read_spikes(0, T), net.state(S.FIELD_ACC), net.stats())
        finally:
            os.environ.pop("SPICE_NO_PERSIST", None)
    for persist, (spk, acc, st) in out.items():
        bad = [t for t in range(T) if not np.array_equal(spk[t], want[t])]
        assert not bad, f"persist={persist}: first mismatching step {bad[0]}"
        assert np.array_equal(acc, o.state(O.F_ACC)), f"persist={persist}: accumulators"
        assert st["fired"] == sum(len(s) for s in want)
        assert st["delivered"] == int(o.delivered().sum())
