"""The PEER spike exchange (device-initiated synchronisation; P:287-290
§III-D/E) executed for real on the GPU, against the G = 1 oracle (partition
invariance):

1. G ranks in one process on cuda:0: every rank's graphs run concurrently on their own
   streams; the update kernels store bitmap words into all windows, the flag kernels
   synchronise them (no host step between ranks).
2. Two processes on cuda:0, each one rank: the windows are CUDA IPC mappings (the same
   path as two GPUs of one box; here the two contexts time-slice the GPU).
3. bench.py under torchrun with two ranks (--same-device), whose in-run oracle check
   (synth spike union + sampled accumulators) must report parity."""
import json
import multiprocessing as mp
import os
import subprocess
import sys

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = {
    "synth20000": (W.synth(20000, 31, 0.005, seed=3), {}, 160),
    "brunel3000_d15": (W.brunel(3000, 0.1, seed=5, delay=15), {}, 160),
    "vogels4000": (W.vogels(4000), dict(tile_width=256), 160),
    "synth20000_cluster2": (W.synth(20000, 31, 0.005, seed=13), dict(tile_width=1024, ctas_per_tile=2), 100),
    "bplus2001": (W.brunel_plus(2001, 0.15, seed=7, delay=3), dict(tile_width=96), 120),
}


@pytest.fixture(scope="module")
def S():
    from paper_2102_04681_b200 import build as B
    B.build()
    from paper_2102_04681_b200 import spice
    return spice


def _oracle(cfg, T):
    o = O.OracleNet(cfg)
    o.step(T)
    return o


def _check(S, cfg, T, G, Sw, results, o):
    want = o.spikes()
    field, ofield = (S.FIELD_ACC, O.F_ACC) if cfg.model == W.SYNTH else (S.FIELD_V, O.F_V)
    full = o.state(ofield)
    fired = delivered = 0
    for g, (spikes, state, stats) in enumerate(results):
        bad = [t for t in range(T) if not np.array_equal(spikes[t], want[t])]
        assert not bad, f"rank {g}: first mismatching step {bad[0]}"
        ids = np.array([S.partition_local_to_global(i, g, G, Sw) for i in range(len(state))])
        assert np.array_equal(state, full[ids]), f"rank {g} state"
        fired += stats["fired"]
        delivered += stats["delivered"]
    assert fired == sum(len(s) for s in want)
    assert delivered == int(o.delivered().sum())


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("name", list(CASES))
def test_peer_exchange_ranks_in_one_process(S, G, name):
    cfg, kw, T = CASES[name]
    Sw = 32
    nets = [S.Network(cfg, rank=g, world_size=G, slice_width=Sw, record_steps=T,
                      exchange=S.EXCHANGE_PEER, **kw) for g in range(G)]
    try:
        with pytest.raises(S.SpiceError):
            nets[0].step(1)                               # not connected yet
        handles = [n.peer_handle() for n in nets]
        for n in nets:
            n.peer_connect(handles)
        for chunk in (1, 20, 64, T - 85):                 # graphs of every size, ranks interleaved
            for n in nets:
                n.step(chunk)
        assert nets[0].stats()["steps"] == T
        field = S.FIELD_ACC if cfg.model == W.SYNTH else S.FIELD_V
        results = [(n.read_spikes(0, T), n.state(field), n.stats()) for n in nets]
    finally:
        for n in nets:
            n.free()
    _check(S, cfg, T, G, Sw, results, _oracle(cfg, T))


def _rank_process(rank, G, name, conn):
    sys.path.insert(0, ROOT)
    from paper_2102_04681_b200 import spice as S2
    cfg, kw, T = CASES[name]
    net = S2.Network(cfg, rank=rank, world_size=G, slice_width=32, record_steps=T,
                     exchange=S2.EXCHANGE_PEER, **kw)
    conn.send(net.peer_handle())
    net.peer_connect(conn.recv())
    net.step(T)
    field = S2.FIELD_ACC if cfg.model == W.SYNTH else S2.FIELD_V
    conn.send((net.read_spikes(0, T), net.state(field), net.stats()))
    net.free()
    conn.close()


@pytest.mark.parametrize("name", ["synth20000", "brunel3000_d15"])
def test_peer_exchange_two_processes_ipc(S, name):
    cfg, _, T = CASES[name]
    G = 2
    ctx = mp.get_context("spawn")
    pipes = [ctx.Pipe() for _ in range(G)]
    procs = [ctx.Process(target=_rank_process, args=(g, G, name, pipes[g][1])) for g in range(G)]
    for p in procs:
        p.start()
    try:
        handles = [pipes[g][0].recv() for g in range(G)]
        for g in range(G):
            pipes[g][0].send(handles)
        results = []
        for g in range(G):
            assert pipes[g][0].poll(600), f"rank {g} did not finish"
            results.append(pipes[g][0].recv())
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    _check(S, cfg, T, G, 32, results, _oracle(cfg, T))


def test_bench_two_ranks_peer_parity(S):
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29561",
                        os.path.join(ROOT, "bench.py"), "--gpus", "2", "--same-device",
                        "--workload", "synth250m", "--scaling", "strong", "--steps", "64", "--warmup", "4",
                        "--profile-steps", "4", "--e2e-steps", "64", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["parity"]["ok"] is True and line["parity"]["ranks"] == 2
    assert line["config"]["exchange"].startswith("device-initiated")


def test_external_exchange_over_host_buffers(S):
    """spice_exchange_get_send / _set_recv: G = 3 virtual ranks whose bitmaps travel through
    host memory (a caller-owned transport) on the fused G > 1 sequence; spike trains equal
    the G = 1 oracle's."""
    cfg, T, G = W.synth(5003, 31, 0.05, seed=23), 40, 3
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    nets = [S.Network(cfg, rank=g, world_size=G, external_exchange=True, record_steps=T)
            for g in range(G)]
    try:
        Wd = nets[0].words_per_rank
        bufs = [np.zeros(Wd, dtype=np.uint32) for _ in range(G)]
        for n in nets:
            n.exchange_begin()
        for t in range(T):
            for g, n in enumerate(nets):
                n.exchange_get_send(bufs[g])
            for n in nets:
                for g in range(G):
                    n.exchange_set_recv(g, bufs[g])
            for n in nets:
                if t < T - 1:
                    n.exchange_end_fused()
                else:
                    n.exchange_end()
        for n in nets:
            got = n.read_spikes(0, T)
            assert all(np.array_equal(a, b) for a, b in zip(got, want))
        with pytest.raises(S.SpiceError):
            nets[0].exchange_set_recv(G, bufs[0])
    finally:
        for n in nets:
            n.free()


def test_compacted_readout_over_ranks(S):
    """Device read-out compaction at G = 2 (global IDs interleaved across the ranks' slices,
    ascending): spice_spikes_prefetch / _collect equal the host decode of spice_read_spikes and
    the G = 1 oracle's spike trains."""
    cfg, T, K, G = W.synth(200_000, 31, 0.004, seed=9), 24, 12, 2
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    nets = [S.Network(cfg, rank=g, world_size=G, slice_width=64, external_exchange=True, record_steps=T)
            for g in range(G)]
    try:
        for _ in range(T):
            for n in nets:
                n.exchange_begin()
            for d in nets:
                for s in nets:
                    d.exchange_put_from(s)
            for n in nets:
                n.exchange_end()
        ids = np.zeros(cfg.n * K, dtype=np.uint32)
        offs = np.zeros(K + 1, dtype=np.uint64)
        for n in nets:
            assert K * G * n.words_per_rank >= 1 << 16           # the compacted path
            for c in range(T // K):
                n.spikes_prefetch(c * K, (c + 1) * K, c & 1)
                n.spikes_collect_into(c & 1, ids, offs)
                for q in range(K):
                    assert np.array_equal(ids[int(offs[q]):int(offs[q + 1])], want[c * K + q]), (c, q)
            assert all(np.array_equal(a, b) for a, b in zip(n.read_spikes(0, T), want))
    finally:
        for n in nets:
            n.free()
