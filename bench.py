#!/usr/bin/env python
"""Benchmark of the Spice hot path on B200 (BASELINE.json metric: synaptic events/s and
wall-clock per 10K steps, whole box, at 1/2/4/8 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload synth|brunel100k|vogels4000]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
    python bench.py --impl reference        # the CPU oracle arm (bounded sample, host cores)

A step = one pass of the whole hot path (neuron update + spike compaction, [all-gather],
delivery) over the network.  Default workload: synth with 3e9 synapses per GPU at the
paper's density 0.156 % and activity 0.5 %, weak scaling (N grows with G).
Timing: W warm-up steps, then exactly K steps between barrier + synchronize, CUDA events on
the library stream, max over ranks.  The synapse stream (12 GB/GPU) is far larger than L2,
so no explicit flush is needed.  One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "synaptic events/sec & wall-clock per 10K steps (whole box) at 1/2/4/8 B200"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", default="spice", choices=["spice", "reference"])
    ap.add_argument("--workload", default="synth",
                    choices=["synth", "synth250m", "brunel100k", "brunelplus50k", "vogels4000"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="synth workloads: weak = fixed synapses per GPU (N grows with G), "
                         "strong = the G=1 network split over G GPUs")
    ap.add_argument("--tile-width", type=int, default=0)
    ap.add_argument("--ctas-per-tile", type=int, default=0)
    ap.add_argument("--global-atomics", action="store_true", help="paper-style delivery (A/B)")
    ap.add_argument("--procedural", action="store_true",
                    help="procedural connectivity (NEXT-4): rows regenerated per spike, none stored (A/B)")
    ap.add_argument("--unfused", action="store_true",
                    help="separate update and delivery launches per step (the G > 1 kernel sequence, A/B)")
    ap.add_argument("--profile-steps", type=int, default=200)
    ap.add_argument("--e2e-steps", type=int, default=1024)
    ap.add_argument("--e2e-chunk", type=int, default=128,
                    help="steps per spice_step call in the e2e leg (every step's spikes are read back, chunk by chunk)")
    ap.add_argument("--no-parity", action="store_true", help="skip the in-run oracle check (synth)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="G > 1 spike exchange: device-initiated stores into peer windows (default) "
                         "or an NCCL all-gather inside the step graph")
    ap.add_argument("--same-device", action="store_true",
                    help="tests only: every rank on cuda:0 (host collectives over gloo)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--setup", action="store_true",
                    help="setup-time experiment (PAPER.md Fig. 9): generator throughput vs size, synth density 5%%")
    return ap.parse_args()


def workload(name: str, G: int, scaling: str = "weak"):
    if name in ("synth", "synth250m"):
        per = 3.0e9 if name == "synth" else 250e6
        tag = "3e9" if name == "synth" else "250m"
        if scaling == "strong":
            return W.synth_for_synapses(per), f"synth_{tag}_synapses_total_strong"
        return W.synth_for_synapses(per * G), f"synth_{tag}_synapses_per_gpu"
    if name == "brunel100k":
        return W.brunel(100_000), "brunel100k"
    if name == "brunelplus50k":
        return W.brunel_plus(50_000), "brunelplus50k"
    return W.vogels(4000), "vogels4000"


def cpu_sample(name: str, cfg):
    """Bounded sample of the workload for the CPU oracle."""
    if name in ("synth", "synth250m"):
        n = cfg.n // 32
        return W.synth(n, cfg.rules[0].k, cfg.activity, cfg.seed), \
            f"synth N={n} (1/32 of the GPU workload's neurons) with the same in-degree K={cfg.rules[0].k} and activity"
    if name == "brunel100k":
        return W.brunel(12_500), "brunel N=12,500 (base scale, p=0.1) instead of 100K"
    if name == "brunelplus50k":
        return W.brunel_plus(6_250), "brunel+ N=6,250 (p=0.1, same STDP) instead of 50K"
    return cfg, "vogels4000 (full workload)"


def ncu_traffic(workload_name: str, delivery: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture
    (profiles/ncu_traffic.json), when it was taken on this workload and tile geometry."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f)[workload_name]
        if e["delivery"] != delivery:
            return None, None
        # a persistent launch runs several steps: traffic per step, like `achieved`
        return float(e["dram_bytes_read"] + e["dram_bytes_write"]) / float(e.get("steps_per_launch", 1)), e["capture"]
    except Exception:
        return None, None


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 9 and p[1].replace(".", "").isdigit():
                rows.append(p)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        load = [float(r[1]) for r in rows if float(r[3]) > 300] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": float(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(rows)}


def run_oracle(cfg, warmup: int, steps: int = 0, seconds: float = 0.0):
    """Time the oracle as it stands (single thread).  Returns events/s, steps, seconds."""
    from oracle import oracle as O
    net = O.OracleNet(cfg)
    net.step(warmup)
    d0 = int(net.delivered().sum()) if net.t else 0
    t0 = time.perf_counter()
    done = 0
    while (steps and done < steps) or (seconds and time.perf_counter() - t0 < seconds) or done == 0:
        net.step(1)
        done += 1
    el = time.perf_counter() - t0
    ev = int(net.delivered().sum()) - d0
    return ev / el, done, el, net.nnz


def main_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, wl = workload(args.workload, args.gpus, args.scaling)
    sample, desc = cpu_sample(args.workload, cfg)
    eps, done, el, nnz = run_oracle(sample, max(3, args.warmup // 10), steps=args.steps)
    line = {"impl": "reference", "metric": METRIC, "value": eps, "unit": "events/s",
            "n_gpus": args.gpus, "steps": done, "warmup": max(3, args.warmup // 10),
            "ms_per_step": el / done * 1e3, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u32" if cfg.model == W.SYNTH else "f32",
            "data": "synthetic", "config": {"workload": wl, "sample": desc, "sample_synapses": nnz},
            "cpu_baseline": {"value": eps, "unit": "events/s", "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": eps, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def parity_check(net, cfg, rank: int, world: int, slice_width: int, n_acc: int = 2):
    """In-run validation against the oracle at the bench size (reading R17):
    (1) the spike union of the last two recorded steps, read through spice_read_spikes
    (every rank decodes the gathered bitmaps of all ranks), equals the synth Bernoulli
    definition; (2) the accumulators of n_acc sampled owned targets equal the brute-force
    sum over their in-synapses of the sources' spike counts.  Synth only (the other
    workloads are checked at full size by tests/test_gpu_fullsize.py)."""
    if cfg.model != W.SYNTH:
        return None
    from oracle import oracle as O
    T = net.stats()["steps"]
    ok = True
    for t in (T - 2, T - 1):
        got = net.read_spikes(t, t + 1)[0]
        ok &= bool(np.array_equal(got, O.synth_fired(cfg, t)))
    acc = net.state(net_field_acc())
    rng = np.random.default_rng(1234 + rank)
    local = rng.choice(net.n_owned, size=min(n_acc, net.n_owned), replace=False)
    for i in local:
        from paper_2102_04681_b200 import spice as S
        j = S.partition_local_to_global(int(i), rank, world, slice_width)
        ok &= O.synth_acc(cfg, j, T) == int(acc[i])
    return {"ok": bool(ok), "steps": T,
            "checked": f"spike union of steps {T - 2}, {T - 1} (all {cfg.n} neurons) vs the Bernoulli "
                       f"definition; accumulators of {len(local)} sampled targets per rank vs the "
                       f"sum over their in-synapses (oracle/spice_oracle.c orc_synth_fired, orc_synth_acc)"}


def net_field_acc():
    from paper_2102_04681_b200 import spice as S
    return S.FIELD_ACC


def main_spice(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2102_04681_b200 import build as B
    if local == 0:                                 # one build per node; the others wait
        B.build()
    if world > 1:
        dist.barrier()
    from paper_2102_04681_b200 import spice as S

    cfg, wl = workload(args.workload, world, args.scaling)
    nccl_id = None
    peer = world > 1 and args.exchange == "peer"
    if world > 1 and not peer:
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    record = max(4 * args.e2e_chunk, 256)
    t0 = time.perf_counter()
    net = S.Network(cfg, rank=rank, world_size=world, device=local, nccl_id=nccl_id,
                    record_steps=record, global_atomics=args.global_atomics,
                    tile_width=args.tile_width, ctas_per_tile=args.ctas_per_tile, unfused=args.unfused,
                    exchange=S.EXCHANGE_PEER if peer else S.EXCHANGE_NCCL, procedural=args.procedural)
    if peer:                                       # map every rank's receive window
        handles = [None] * world
        dist.all_gather_object(handles, net.peer_handle())
        net.peer_connect(handles)
    setup_s = time.perf_counter() - t0
    info = net.info()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allreduce(x, op):
        if world == 1:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device="cpu" if args.same_device else "cuda")
        dist.all_reduce(t, op=op)
        return t.item()

    MAX = dist.ReduceOp.MAX if world > 1 else None
    SUM = dist.ReduceOp.SUM if world > 1 else None
    MIN = dist.ReduceOp.MIN if world > 1 else None

    # ---- warm-up ----
    net.step(args.warmup)
    net.sync()
    barrier()
    s0 = net.stats()
    clocks = ClockSampler(local)
    clocks.start()
    stream = torch.cuda.ExternalStream(net.stream)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    net.step(args.steps)
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    ck = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    s1 = net.stats()
    ms_max = allreduce(ms, MAX)
    events = allreduce(s1["delivered"] - s0["delivered"], SUM)
    fired = allreduce(s1["fired"] - s0["fired"], SUM)
    value = events / (ms_max / 1e3)
    launches = net.launches(args.steps)

    # ---- per-kernel live timing for the roofline (CUDA events on the library stream) ----
    prof = net.profile(args.profile_steps)
    ev_step = events / args.steps / world     # per launch of this rank's step kernel
    sp_step = fired / args.steps
    # 4 B target record per event + 12 B per spike (row pointer + list entry)
    bytes_launch = 4.0 * ev_step + 12.0 * sp_step
    peak, peak_src = hbm_peak()
    fused = prof["fused"] > 0
    small = net.launches(32) == 2                  # one-CTA persistent kernel (small networks)
    persistent = net.launches(32) == 4             # persistent synth kernel: one launch per replay
    kern = ("k_small (whole steps, one CTA, 32 per launch)" if small else
            "persistent step kernel (k_synth_run: the steps of a replay in one launch, "
            "deliver t + update/publish t+1 per step, grid barrier between steps; time per step)" if persistent else
            "k_fused (deliver t + update t+1)") if fused else ("k_global_atomics" if args.global_atomics else "k_deliver")
    # spice_step runs the fused kernel back to back inside captured graphs: the in-graph
    # timing is the kernel as the timed region ran it (the individually launched timing
    # carries launch overhead the graph does not)
    launch_ms = (prof["fused_in_graph"] or prof["fused"]) if fused else prof["deliver"]
    achieved = bytes_launch / (launch_ms * 1e-3) / 1e9
    step_ms = ms_max / args.steps

    # ---- end to end through the public API: steps in chunks, every step's spikes read
    #      back to host memory (double-buffered: chunk c's copy and decode overlap chunk c+1)
    G, Sw = world, net.slice_width
    words = S.partition_owned_count(cfg.n, 0, G, Sw)
    d2h = G * ((words + 31) // 32) * 4
    K = args.e2e_chunk
    nchunks = max(1, args.e2e_steps // K)
    ids = np.zeros(cfg.n * K // 8 + 1024, dtype=np.uint32)
    offs = np.zeros(K + 1, dtype=np.uint64)
    t_now = net.stats()["steps"]
    for c in range(2):                              # untimed: allocates both pinned slots
        net.step(K)
        net.spikes_prefetch(t_now + c * K, t_now + (c + 1) * K, c)
    for c in range(2):
        net.spikes_collect_into(c, ids, offs)
    t_now += 2 * K
    got_spikes = 0
    barrier()
    te = time.perf_counter()
    for c in range(nchunks):
        net.step(K)
        net.spikes_prefetch(t_now + c * K, t_now + (c + 1) * K, c & 1)
        if c:
            got_spikes += net.spikes_collect_into((c - 1) & 1, ids, offs)
    got_spikes += net.spikes_collect_into((nchunks - 1) & 1, ids, offs)
    e2e_s = time.perf_counter() - te
    barrier()
    e2e_s = allreduce(e2e_s, MAX)
    e2e_events = events / args.steps * nchunks * K     # same per-step work
    e2e_value = e2e_events / e2e_s
    compacted = K * G * ((words + 31) // 32) >= (1 << 16)
    if compacted:   # device-compacted read-out: counts + the IDs guess (1.25 x the last chunk + 4096)
        d2h = int(4 + 4 * (1.25 * got_spikes / (nchunks * K) + 4096 / K))

    parity = None
    if not args.no_parity:
        p = parity_check(net, cfg, rank, world, Sw)
        if p is not None:
            p["ok"] = bool(allreduce(1.0 if p["ok"] else 0.0, MIN) > 0.5)
            p["ranks"] = world
            parity = p

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        sample, desc = cpu_sample(args.workload, cfg)
        if world > 1:
            desc += f" (sample of the whole {world}-GPU network)"
        eps, done, el, _ = run_oracle(sample, 3, seconds=args.cpu_seconds)
        cpu = {"value": eps, "unit": "events/s", "cores": 1, "kind": "oracle",
               "sample": f"{desc}; {done} steps in {el:.1f} s, single thread"}

    delivery = ("procedural: row segments regenerated per spike and tile from Philox, no adjacency stored"
                if args.procedural else
                "global-atomics (paper-style A/B)" if args.global_atomics else
                f"one CTA, {info['tile_width']} targets in smem, 32 steps per launch" if small else
                f"tiled smem, {info['n_tiles']} tiles x {info['tile_width']} targets, {info['ctas_per_tile']} CTA/tile")
    traffic, traffic_src = ncu_traffic(wl, delivery) if fused else (None, None)
    line = {
        "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "wall_s_per_10k_steps": step_ms * 10.0,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "u32" if cfg.model == W.SYNTH else "f32",
        "data": "synthetic (seeded Philox network and drive; no datasets)",
        "config": {"workload": wl, "n_neurons": cfg.n,
                   "in_degree": cfg.rules[0].k if cfg.model == W.SYNTH else None,
                   "activity": cfg.activity if cfg.model == W.SYNTH else None, "delay": cfg.delay,
                   "synapses_total": int(allreduce(info["n_synapses"], SUM)),
                   "synapses_rank0": info["n_synapses"], "spikes_per_step": fired / args.steps,
                   "events_per_step": events / args.steps,
                   "parallelism": f"model-parallel strided neuron slices x{world}",
                   "exchange": (None if world == 1 else
                                "device-initiated: update kernel stores bitmap words into every rank's window, "
                                "flag release/acquire kernels (no host round trip)" if peer else
                                "NCCL all-gather of spike bitmaps in the step graph"),
                   "delivery": delivery,
                   "l2": "no flush: synapse stream per step >> 126 MB L2 is read from 12 GB/GPU",
                   "setup_s": setup_s},
        "roofline": {"bound": "hbm", "kernel": kern, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "bytes_per_launch": bytes_launch, "launch_ms": launch_ms,
                     "bytes_model": "SURVEY §8(d): 4 B/event + 12 B/spike (delivery bytes only), rank 0's share",
                     "peak_source": peak_src,
                     "kernel_share_of_step": launch_ms / step_ms if fused else None,
                     "kernel_ms": prof},
        "e2e": {"value": e2e_value, "unit": "events/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": d2h, "steps": nchunks * K, "spikes_read": got_spikes,
                "note": (f"spice_step({K}) + spice_spikes_prefetch of those steps: bitmaps compacted into "
                         f"ascending spike IDs on the device, counts and IDs copied to pinned host memory, "
                         f"spice_spikes_collect fills the caller's arrays while the next chunk runs (double-buffered)"
                         if compacted else
                         f"spice_step({K}) + spice_spikes_prefetch of those steps' bitmaps to pinned host memory, "
                         f"decoded by spice_spikes_collect while the next chunk runs (double-buffered)")},
        "gpu_launches": launches,
        "clocks": ck,
        "parity": parity,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    net.free()
    if world > 1:
        dist.destroy_process_group()
    return 0


SETUP_SIZES = (4_000, 16_000, 64_000, 128_000, 245_000)   # 0.8M .. 3.0e9 synapses at density 5 %


def main_setup(args):
    """Setup time vs network size (Fig. 9: Synth, density 5 %; P:443:
    "our actual setup kernel generates networks at ~200M synapses/ms").  Two rules at each
    size: the synth fixed in-degree rule K = 0.05 N (reading R9) and the paper's Bernoulli
    descriptor {range, range, p = 0.05}.  gen_ms = device time of the generator
    kernels; create_ms = host wall time of spice_create_network (allocation, generation,
    state init, graph capture), each the median of `reps` creations after one warm-up."""
    import torch
    torch.cuda.set_device(0)
    from paper_2102_04681_b200 import build as B
    B.build()
    from paper_2102_04681_b200 import spice as S
    points = []
    reps = 3
    for n in SETUP_SIZES:
        k = round(0.05 * n)
        for kind, cfg in (("fixed_indegree", W.NetConfig(f"setup_indeg{n}", W.SYNTH, n, n,
                                                          (W.Rule((0, n), (0, n), W.FIXED_INDEGREE, k=k),),
                                                          0.1, 1, 1, 0.005, ())),
                          ("fixed_prob", W.NetConfig(f"setup_prob{n}", W.SYNTH, n, n,
                                                      (W.Rule((0, n), (0, n), W.FIXED_PROB, p=0.05),),
                                                      0.1, 1, 1, 0.005, ()))):
            gens, walls, syn = [], [], 0
            for r in range(reps + 1):
                with S.Network(cfg, record_steps=8) as net:
                    t = net.setup_times()
                    syn = net.info()["n_synapses"]
                if r:
                    gens.append(t["gen_ms"])
                    walls.append(t["create_ms"])
            g, w = statistics.median(gens), statistics.median(walls)
            points.append({"n_neurons": n, "rule": kind, "synapses": syn, "gen_ms": g, "create_ms": w,
                           "gen_synapses_per_ms": syn / g if g else None,
                           "create_synapses_per_ms": syn / w if w else None})
            print(f"setup n={n} {kind}: {syn:.3e} synapses, generator {g:.2f} ms ({syn / g / 1e6:.1f}M syn/ms), "
                  f"create {w:.1f} ms", file=sys.stderr, flush=True)
    best = max(p["gen_synapses_per_ms"] for p in points if p["gen_synapses_per_ms"])
    line = {"metric": "setup: synapses generated per ms (generator kernels), synth density 5 %",
            "value": best, "unit": "synapses/ms", "higher_is_better": True, "n_gpus": 1,
            "data": "synthetic", "paper_context": "~200M synapses/ms on V100 (PAPER.md:443)",
            "config": {"workload": "setup_synth_density5pct", "sizes": list(SETUP_SIZES), "reps": reps},
            "points": points}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse_args()
    if args.setup:
        return main_setup(args)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return main_reference(args)
    return main_spice(args)


if __name__ == "__main__":
    sys.exit(main())
