"""ctypes front-end of the CPU oracle (oracle/spice_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py, never by the product package
``paper_2102_04681_b200``.  It depends only on ``workloads`` (inputs) and numpy.

Two builds of the same C source: ``mirror32`` (fp32, the paper's single precision,
PAPER.md:436) and ``ref64`` (fp64, for closed-form pins).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spice_oracle.c")
_BUILD = os.path.join(_HERE, "build")

VOGELS, BRUNEL, BRUNEL_PLUS, SYNTH = 1, 2, 3, 4
F_V, F_GE, F_GI, F_REF, F_ACC, F_XTR, F_YTR = range(7)


def build(force: bool = False) -> None:
    """Compile both oracle variants with gcc (-ffp-contract=off: no fused multiply-add)."""
    os.makedirs(_BUILD, exist_ok=True)
    for tag, real in (("32", "float"), ("64", "double")):
        out = os.path.join(_BUILD, f"liboracle{tag}.so")
        if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(_SRC):
            continue
        cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-fvisibility=hidden", f"-DORC_REAL={real}", "-o", out + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(out + ".tmp", out)


class _Rule(C.Structure):
    _fields_ = [("src_begin", C.c_uint32), ("src_end", C.c_uint32),
                ("dst_begin", C.c_uint32), ("dst_end", C.c_uint32),
                ("kind", C.c_uint32), ("k", C.c_uint32), ("plastic", C.c_uint32),
                ("delay_min", C.c_uint16), ("delay_max", C.c_uint16), ("p", C.c_double)]


_LIBS = {}


def lib(precision: str = "mirror32"):
    tag = {"mirror32": "32", "ref64": "64"}[precision]
    if tag in _LIBS:
        return _LIBS[tag]
    build()
    L = C.CDLL(os.path.join(_BUILD, f"liboracle{tag}.so"))
    vp, u32, u64, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_double
    L.orc_create.restype = vp
    L.orc_create.argtypes = [u32, u32, u32, C.POINTER(_Rule), u32, dbl, u32, u64, dbl,
                             C.POINTER(C.c_double), u32, u32, u32, u32]
    L.orc_free.argtypes = [vp]
    L.orc_step.argtypes = [vp, u64]
    L.orc_nnz.restype = u64; L.orc_nnz.argtypes = [vp]
    L.orc_time.restype = u64; L.orc_time.argtypes = [vp]
    for f in ("orc_row_ptr", "orc_targets", "orc_plastic_flags", "orc_spike_offsets",
              "orc_spikes_all", "orc_delivered"):
        getattr(L, f).argtypes = [vp, vp]
    L.orc_weights.argtypes = [vp, vp]
    L.orc_spike_count_total.restype = u64; L.orc_spike_count_total.argtypes = [vp]
    L.orc_get_state.argtypes = [vp, u32, vp]
    L.orc_set_state.argtypes = [vp, u32, vp]
    L.orc_get_input.argtypes = [vp, u32, vp, vp]
    L.orc_force_next.argtypes = [vp, vp, u64, C.c_int]
    L.orc_philox.argtypes = [vp, vp, vp]
    L.orc_poisson_table.restype = u32; L.orc_poisson_table.argtypes = [dbl, vp, u32]
    L.orc_owner.restype = u32; L.orc_owner.argtypes = [u64, u32, u32]
    L.orc_local_to_global.restype = u64; L.orc_local_to_global.argtypes = [u64, u32, u32, u32]
    L.orc_sizeof_real.restype = u32
    L.orc_row.restype = u64
    L.orc_row.argtypes = [C.POINTER(_Rule), u32, u64, u32, u32, u32, u32, vp, u64]
    L.orc_col.restype = u64
    L.orc_col.argtypes = [C.POINTER(_Rule), u32, u64, u32, vp, u64]
    L.orc_synth_fired.restype = u64
    L.orc_synth_fired.argtypes = [u32, dbl, u64, u64, vp, u64]
    L.orc_synth_acc.restype = u64
    L.orc_synth_acc.argtypes = [C.POINTER(_Rule), u32, u64, dbl, u32, u64, u32]
    L.orc_delays.argtypes = [vp, vp]
    L.orc_ring_slots.restype = u32; L.orc_ring_slots.argtypes = [vp]
    L.orc_set_input.argtypes = [vp, u32, vp]
    L.orc_set_time.argtypes = [vp, u64]
    _LIBS[tag] = L
    return L


def philox(ctr: Sequence[int], key: Sequence[int]) -> np.ndarray:
    L = lib()
    c = np.asarray(ctr, dtype=np.uint32); k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    L.orc_philox(c.ctypes.data, k.ctypes.data, o.ctypes.data)
    return o


def poisson_table(lam: float) -> np.ndarray:
    out = np.zeros(1024, dtype=np.uint64)
    n = lib().orc_poisson_table(lam, out.ctypes.data, 1024)
    return out[:n]


def _rules(cfg):
    rules = (_Rule * max(1, len(cfg.rules)))()
    for i, r in enumerate(cfg.rules):
        rules[i] = _Rule(r.src[0], r.src[1], r.dst[0], r.dst[1], r.kind, r.k, 1 if r.plastic else 0,
                         r.delay_min, r.delay_max, float(r.p))
    return rules


def row(cfg, s: int, part: Optional[tuple] = None) -> np.ndarray:
    """Sorted targets of source s (brute force, no network built)."""
    g, G, S = part if part else (0, 1, 1)
    cap = 1 << 16
    while True:
        out = np.zeros(cap, dtype=np.uint32)
        n = lib().orc_row(_rules(cfg), len(cfg.rules), cfg.seed, s, g, G, S, out.ctypes.data, cap)
        if n <= cap:
            return out[:n]
        cap = int(n)


def col(cfg, j: int) -> np.ndarray:
    """Sorted sources (with multiplicity) of all edges into target j."""
    cap = 1 << 16
    while True:
        out = np.zeros(cap, dtype=np.uint32)
        n = lib().orc_col(_rules(cfg), len(cfg.rules), cfg.seed, j, out.ctypes.data, cap)
        if n <= cap:
            return out[:n]
        cap = int(n)


def synth_fired(cfg, t: int) -> np.ndarray:
    """Synth spike set of step t by the Bernoulli definition (reading R12), no simulation."""
    out = np.zeros(max(16, int(cfg.n * cfg.activity * 2) + 64), dtype=np.uint32)
    while True:
        n = lib().orc_synth_fired(cfg.n, cfg.activity, cfg.seed, t, out.ctypes.data, out.size)
        if n <= out.size:
            return out[:n]
        out = np.zeros(int(n), dtype=np.uint32)


def synth_acc(cfg, j: int, T: int) -> int:
    """Synth accumulator of target j after T steps (sampled-column check, reading R17)."""
    return int(lib().orc_synth_acc(_rules(cfg), len(cfg.rules), cfg.seed, cfg.activity, j, T, cfg.delay))


def owner(j: int, G: int, S: int) -> int:
    return lib().orc_owner(j, G, S)


def local_to_global(i: int, g: int, G: int, S: int) -> int:
    return lib().orc_local_to_global(i, g, G, S)


class OracleNet:
    """One oracle network.  ``cfg`` is a :class:`workloads.NetConfig`.
    ``part=(g, G, S)`` keeps only targets owned by rank g."""

    def __init__(self, cfg, precision: str = "mirror32", part: Optional[tuple] = None):
        self.cfg = cfg
        self.L = lib(precision)
        self.real = np.float32 if precision == "mirror32" else np.float64
        rules = (_Rule * max(1, len(cfg.rules)))()
        for i, r in enumerate(cfg.rules):
            rules[i] = _Rule(r.src[0], r.src[1], r.dst[0], r.dst[1], r.kind, r.k,
                             1 if r.plastic else 0, r.delay_min, r.delay_max, float(r.p))
        prm = (C.c_double * max(1, len(cfg.params)))(*cfg.params)
        g, G, S = part if part else (0, 1, 1)
        self.h = self.L.orc_create(cfg.model, cfg.n, cfg.n_exc, rules, len(cfg.rules),
                                   cfg.dt_ms, cfg.delay, cfg.seed, cfg.activity,
                                   prm, len(cfg.params), g, G, S)
        if not self.h:
            raise ValueError("oracle rejected the configuration")
        self.n = cfg.n

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.L.orc_free(h)
            self.h = None

    # connectivity -----------------------------------------------------------
    @property
    def nnz(self) -> int:
        return self.L.orc_nnz(self.h)

    def csr(self):
        rp = np.zeros(self.n + 1, dtype=np.uint64)
        self.L.orc_row_ptr(self.h, rp.ctypes.data)
        tg = np.zeros(max(1, self.nnz), dtype=np.uint32)
        self.L.orc_targets(self.h, tg.ctypes.data)
        return rp, tg[: self.nnz]

    def delays(self) -> np.ndarray:
        """Per-synapse delays in CSR order (reading R19)."""
        d = np.zeros(max(1, self.nnz), dtype=np.uint16)
        self.L.orc_delays(self.h, d.ctypes.data)
        return d[: self.nnz]

    @property
    def ring_slots(self) -> int:
        return self.L.orc_ring_slots(self.h)

    def plastic_flags(self) -> np.ndarray:
        f = np.zeros(max(1, self.nnz), dtype=np.uint8)
        self.L.orc_plastic_flags(self.h, f.ctypes.data)
        return f[: self.nnz]

    def weights(self) -> np.ndarray:
        w = np.zeros(max(1, self.nnz), dtype=self.real)
        if self.L.orc_weights(self.h, w.ctypes.data) != 0:
            raise ValueError("no plastic weights")
        return w[: self.nnz]

    # simulation -------------------------------------------------------------
    def step(self, n_steps: int) -> None:
        self.L.orc_step(self.h, n_steps)

    @property
    def t(self) -> int:
        return self.L.orc_time(self.h)

    def spikes(self):
        """List over steps of ascending global spike IDs."""
        T = self.t
        off = np.zeros(T + 1, dtype=np.uint64)
        self.L.orc_spike_offsets(self.h, off.ctypes.data)
        tot = self.L.orc_spike_count_total(self.h)
        sp = np.zeros(max(1, tot), dtype=np.uint32)
        self.L.orc_spikes_all(self.h, sp.ctypes.data)
        return [sp[int(off[t]):int(off[t + 1])].copy() for t in range(T)]

    def delivered(self) -> np.ndarray:
        d = np.zeros(max(1, self.t), dtype=np.uint64)
        self.L.orc_delivered(self.h, d.ctypes.data)
        return d[: self.t]

    def state(self, field: int) -> np.ndarray:
        dt = np.uint32 if field in (F_REF, F_ACC) else self.real
        out = np.zeros(self.n, dtype=dt)
        if self.L.orc_get_state(self.h, field, out.ctypes.data) != 0:
            raise ValueError(field)
        return out

    def set_state(self, field: int, values) -> None:
        dt = np.uint32 if field in (F_REF, F_ACC) else self.real
        a = np.ascontiguousarray(values, dtype=dt)
        assert a.shape == (self.n,)
        if self.L.orc_set_state(self.h, field, a.ctypes.data) != 0:
            raise ValueError(field)

    def input(self, rel: int = 0):
        c = np.zeros(self.n, dtype=np.uint32)
        p = np.zeros(self.n, dtype=np.int64)
        if self.L.orc_get_input(self.h, rel, c.ctypes.data, p.ctypes.data) != 0:
            raise ValueError(rel)
        return c, p

    def set_input(self, rel: int, counts) -> None:
        a = np.ascontiguousarray(counts, dtype=np.uint32)
        assert a.shape == (self.n,)
        if self.L.orc_set_input(self.h, rel, a.ctypes.data) != 0:
            raise ValueError(rel)

    def set_time(self, t: int) -> None:
        self.L.orc_set_time(self.h, t)

    def force_next(self, ids, mode: str = "replace") -> None:
        a = np.ascontiguousarray(ids, dtype=np.uint32)
        m = {"replace": 1, "add": 2}[mode]
        if self.L.orc_force_next(self.h, a.ctypes.data, a.size, m) != 0:
            raise ValueError("bad id")
