"""Weak-scaling timing proxy on ONE B200: rank 0's slice of the synth
configuration at 3e9 synapses per GPU for G ranks.  The receive buffer is filled once with
G copies of rank 0's own step bitmap (spice_exchange_get_send / _set_recv; the same spike
count per rank and the same Bernoulli statistics as the real peers' bitmaps, bits past a
rank's owned neurons ignored), then the fused G > 1 step sequence (bitmap->list +
descriptors, fused delivery + update, advance) is captured K times in a CUDA graph and
timed.  Timing only: the peers' bitmaps repeat every step and the exchange is not timed.
Usage: python tools/g_proxy.py G[:C[:TW]] ...   (C = CTAs per tile, TW = tile width; auto if absent)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
PHASES = os.environ.get("SPICE_PHASES") == "1"
if PHASES and "SPICE_LIB" not in os.environ:         # phase clocks: a diagnostic library variant
    import importlib.util  # noqa: E402
    _spec = importlib.util.spec_from_file_location(
        "_spice_build", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2102_04681_b200", "build.py"))
    _B = importlib.util.module_from_spec(_spec)
    _spec.loader.exec_module(_B)
    _B.build(out="/tmp/libspice_phases.so", defines=["SPICE_PHASES_BUILD=1"])
    os.environ["SPICE_LIB"] = "/tmp/libspice_phases.so"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2102_04681_b200 import spice as S  # noqa: E402

K, R = 32, int(os.environ.get("PROXY_R", "20"))
for arg in sys.argv[1:] or ["2", "4", "8"]:
    f = [int(x) for x in arg.split(":")]
    G = f[0]
    kw = {}
    if len(f) > 1 and f[1]:
        kw["ctas_per_tile"] = f[1]
    if len(f) > 2 and f[2]:
        kw["tile_width"] = f[2]
    cfg = W.synth_weak(G)
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    try:
        net = S.Network(cfg, rank=0, world_size=G, external_exchange=True, record_steps=64,
                        stream=s.cuda_stream, **kw)
    except S.SpiceError as e:
        print(json.dumps({"G": G, "args": arg, "error": str(e)}), flush=True)
        continue
    buf = np.zeros(net.words_per_rank, dtype=np.uint32)
    with torch.cuda.stream(s):
        net.exchange_begin()
        for _ in range(8):                       # a few real steps, then freeze the gather
            net.exchange_get_send(buf)
            for r in range(G):
                net.exchange_set_recv(r, buf)
            net.exchange_end_fused()
        net.sync()
        nsp = int(sum(bin(int(x)).count("1") for x in buf)) * G
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(K):
                net.exchange_end_fused()
        for _ in range(3):
            g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(R):
            g.replay()
        e1.record(s)
        s.synchronize()
    ms = e0.elapsed_time(e1) / (R * K)
    if PHASES:
        p = net.debug_phases().astype(np.float64)
        launches = np.maximum(p[:, 13], 1)
        mhz = float(os.environ.get("SM_MHZ", "1965"))
        print("  phases (mean us from CTA start):",
              {sl: round(float((p[:, sl] / launches / mhz).mean()), 2) for sl in range(1, 13) if p[:, sl].any()})
    info = net.info()
    print(json.dumps({"G": G, "args": arg, "n": cfg.n, "k": cfg.rules[0].k, "n_owned": info["n_owned"],
                      "synapses_rank0": info["n_synapses"], "spikes_per_step": nsp, "tiles": info["n_tiles"],
                      "tile_width": info["tile_width"], "ctas_per_tile": info["ctas_per_tile"],
                      "us_per_step_rank0": round(ms * 1e3, 3)}), flush=True)
    net.free()
    del g
    torch.cuda.empty_cache()
