"""compute-sanitizer driver (diagnostics): small networks that exercise every
step-kernel family -- synth fast path (fire warps, named barriers), 2- and 4-CTA cluster tiles
(DSMEM reductions, cluster barriers), Brunel delta = 15 (update overlapped with delivery), per-synapse
delays, Brunel+ (shared fixed-point sums, lazy STDP), the one-CTA small-network kernel, the
paper-style global-atomics kernel, procedural delivery and two PEER ranks in one process --
a few steps each, then a synchronising read.  Each case checks its spikes against the oracle.

    compute-sanitizer --tool racecheck python tools/sanitize.py [case ...]
"""
import dataclasses
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2102_04681_b200 import spice as S  # noqa: E402


def _delays(cfg, lo, hi):
    return dataclasses.replace(cfg, rules=tuple(dataclasses.replace(r, delay_min=lo, delay_max=hi) for r in cfg.rules))


CASES = {
    "synth_fast_c2": (W.synth(40000, 31, 0.005, seed=12), dict(tile_width=20480, ctas_per_tile=2), 8),
    "synth_c1": (W.synth(20000, 31, 0.005, seed=3), dict(tile_width=4096), 8),
    "synth_c4": (W.synth(20000, 31, 0.005, seed=13), dict(ctas_per_tile=4), 8),
    "brunel_d15": (W.brunel(3000, 0.1, seed=5, delay=15), dict(tile_width=256), 20),
    "brunel_d15_c4": (W.brunel(3000, 0.1, seed=14, delay=15), dict(tile_width=256, ctas_per_tile=4), 20),
    "brunel_delays": (_delays(W.brunel(3000, 0.1, seed=6, delay=2), 2, 9), dict(tile_width=256), 20),
    "brunelplus": (W.brunel_plus(2000, 0.1, seed=7), dict(tile_width=256), 20),
    "vogels_small": (W.vogels(4000), {}, 40),
    "vogels_global_atomics": (W.vogels(4000, seed=9), dict(global_atomics=True), 10),
    "brunel_procedural": (W.brunel(3000, 0.1, seed=5, delay=15), dict(tile_width=256, procedural=True), 20),
}


def run(name):
    cfg, kw, T = CASES[name]
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    with S.Network(cfg, record_steps=T, **kw) as net:
        net.step(T)
        got = net.read_spikes(0, T)
    ok = all(np.array_equal(got[t], want[t]) for t in range(T))
    print(f"{name}: {T} steps, {sum(len(s) for s in want)} spikes, oracle match {ok}", flush=True)
    return ok


def run_peer():
    cfg, T, G = W.synth(20000, 31, 0.005, seed=3), 8, 2
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    nets = [S.Network(cfg, rank=g, world_size=G, slice_width=32, record_steps=T, exchange=S.EXCHANGE_PEER)
            for g in range(G)]
    try:
        hs = [n.peer_handle() for n in nets]
        for n in nets:
            n.peer_connect(hs)
        for n in nets:
            n.step(T)
        got = [n.read_spikes(0, T) for n in nets]
    finally:
        for n in nets:
            n.free()
    ok = all(np.array_equal(g[t], want[t]) for g in got for t in range(T))
    print(f"peer_G2: {T} steps, oracle match {ok}", flush=True)
    return ok


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES) + ["peer_G2"]
    res = [run_peer() if n == "peer_G2" else run(n) for n in names]
    print("all cases match the oracle" if all(res) else "MISMATCH")
