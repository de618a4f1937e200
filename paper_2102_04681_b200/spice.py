"""Thin ctypes binding of libspice.so (include/spice.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no CPU
fallback: if the library is missing or no GPU is visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# SPICE_LIB: alternative build of the same library (used only for A/B experiments)
LIB_PATH = os.environ.get("SPICE_LIB") or os.path.join(_PKG, "libspice.so")

OK, EINVAL, ENOMEM, ECUDA, ENCCL, ERANGE, ETRUNC, ESTATE = range(8)
VOGELS, BRUNEL, BRUNEL_PLUS, SYNTH = 1, 2, 3, 4
FLAG_EXTERNAL_EXCHANGE, FLAG_GLOBAL_ATOMICS, FLAG_UNFUSED, FLAG_USER_STREAM, FLAG_PROCEDURAL = 0x1, 0x2, 0x4, 0x8, 0x10
EXCHANGE_NCCL, EXCHANGE_PEER = 0, 1
FIELD_V, FIELD_GE, FIELD_GI, FIELD_REF, FIELD_ACC, FIELD_XTR, FIELD_YTR = range(7)
ABI_VERSION = 2


class SpiceError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class Rule(C.Structure):
    _fields_ = [("src_begin", C.c_uint32), ("src_end", C.c_uint32),
                ("dst_begin", C.c_uint32), ("dst_end", C.c_uint32),
                ("kind", C.c_uint32), ("k", C.c_uint32), ("plastic", C.c_uint32),
                ("delay_min", C.c_uint16), ("delay_max", C.c_uint16), ("p", C.c_double)]


class Config(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("model", C.c_uint32),
                ("n_neurons", C.c_uint32), ("n_exc", C.c_uint32),
                ("rules", C.POINTER(Rule)), ("n_rules", C.c_uint32),
                ("delay_steps", C.c_uint32), ("dt_ms", C.c_double), ("seed", C.c_uint64),
                ("activity", C.c_double), ("model_params", C.POINTER(C.c_double)),
                ("n_model_params", C.c_uint32), ("rank", C.c_uint32), ("world_size", C.c_uint32),
                ("slice_width", C.c_uint32), ("device", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("record_steps", C.c_uint32), ("flags", C.c_uint32), ("tile_width", C.c_uint32),
                ("ctas_per_tile", C.c_uint32), ("exchange", C.c_uint32),
                ("stream", C.c_void_p), ("dev_alloc", C.c_void_p), ("dev_free", C.c_void_p),
                ("alloc_ctx", C.c_void_p)]


# device allocator callbacks (spice_config.dev_alloc / dev_free)
DEV_ALLOC = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
DEV_FREE = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


_lib = None


def lib():
    """Load libspice.so (fails loudly when it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2102_04681_b200.build`")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    st = C.c_int
    sigs = {
        "spice_create_network": (st, [C.POINTER(Config), C.POINTER(vp)]),
        "spice_step": (st, [vp, u64]),
        "spice_read_spikes": (st, [vp, u64, u64, vp, u64, vp, C.POINTER(u64)]),
        "spice_free": (st, [vp]),
        "spice_spikes_prefetch": (st, [vp, u64, u64, u32]),
        "spice_spikes_collect": (st, [vp, u32, vp, u64, vp, C.POINTER(u64)]),
        "spice_read_connectivity": (st, [vp, u32, u32, vp, u64, vp, C.POINTER(u64)]),
        "spice_read_state": (st, [vp, u32, vp, u64]),
        "spice_write_state": (st, [vp, u32, vp, u64]),
        "spice_read_input": (st, [vp, u32, vp, vp, u64]),
        "spice_read_weights": (st, [vp, u32, u32, vp, u64, C.POINTER(u64)]),
        "spice_read_delays": (st, [vp, u32, u32, vp, u64, C.POINTER(u64)]),
        "spice_force_spikes": (st, [vp, vp, u64, i32]),
        "spice_stats": (st, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
        "spice_stream": (vp, [vp]),
        "spice_sync": (st, [vp]),
        "spice_info": (st, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u32), C.POINTER(u32),
                            C.POINTER(u32), C.POINTER(u64)]),
        "spice_kernels_per_step": (u32, [vp]),
        "spice_launches": (u64, [vp, u64]),
        "spice_setup_times": (st, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "spice_debug_phases": (st, [vp, vp, u64, C.POINTER(u64)]),
        "spice_profile": (st, [vp, u64, vp, u32, C.POINTER(u32)]),
        "spice_last_error": (C.c_char_p, []),
        "spice_nccl_unique_id": (st, [vp]),
        "spice_exchange_begin": (st, [vp]),
        "spice_exchange_end": (st, [vp]),
        "spice_exchange_end_fused": (st, [vp]),
        "spice_exchange_put": (st, [vp, vp]),
        "spice_exchange_get_send": (st, [vp, vp, i32]),
        "spice_exchange_set_recv": (st, [vp, u32, vp, i32]),
        "spice_peer_handle": (st, [vp, vp]),
        "spice_peer_connect": (st, [vp, vp]),
        "spice_partition_owner": (u32, [u64, u32, u32]),
        "spice_partition_local_to_global": (u64, [u64, u32, u32, u32]),
        "spice_partition_owned_count": (u64, [u64, u32, u32, u32]),
        "spice_default_slice_width": (u32, [u64, u32]),
        "spice_decode_bitmaps": (st, [vp, u32, u32, u32, vp, u64, C.POINTER(u64)]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def _ptr(buf) -> int:
    """Address of a numpy array, a torch tensor or a raw integer pointer."""
    if isinstance(buf, int):
        return buf
    if isinstance(buf, np.ndarray):
        return buf.ctypes.data
    return buf.data_ptr()


def _check(status: int) -> None:
    if status != OK:
        raise SpiceError(status, lib().spice_last_error().decode())


# ------------------------------------------------------------- host-only helpers
def partition_owner(j: int, world_size: int, slice_width: int) -> int:
    return lib().spice_partition_owner(j, world_size, slice_width)


def partition_local_to_global(i: int, rank: int, world_size: int, slice_width: int) -> int:
    return lib().spice_partition_local_to_global(i, rank, world_size, slice_width)


def partition_owned_count(n: int, rank: int, world_size: int, slice_width: int) -> int:
    return lib().spice_partition_owned_count(n, rank, world_size, slice_width)


def default_slice_width(n: int, world_size: int) -> int:
    return lib().spice_default_slice_width(n, world_size)


def decode_bitmaps(words: np.ndarray, world_size: int, words_per_rank: int, slice_width: int) -> np.ndarray:
    """Gathered per-rank spike bitmaps of one step -> ascending global IDs (host only)."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    total = C.c_uint64(0)
    out = np.zeros(max(1, int(sum(bin(int(x)).count("1") for x in w))), dtype=np.uint32)
    _check(lib().spice_decode_bitmaps(w.ctypes.data, world_size, words_per_rank, slice_width,
                                      out.ctypes.data, out.size, C.byref(total)))
    return out[: total.value]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().spice_nccl_unique_id(buf))
    return buf.raw


class Network:
    """One rank's slice of a network (``spice_net``).

    ``cfg`` is any object with the fields of ``workloads.NetConfig`` (model, n, n_exc,
    rules, dt_ms, delay, seed, activity, params)."""

    def __init__(self, cfg, rank: int = 0, world_size: int = 1, slice_width: int = 0,
                 device: int = 0, record_steps: int = 1024, nccl_id: Optional[bytes] = None,
                 external_exchange: bool = False, global_atomics: bool = False,
                 tile_width: int = 0, ctas_per_tile: int = 0, unfused: bool = False,
                 exchange: int = EXCHANGE_NCCL, stream: Optional[int] = None,
                 allocator=None, procedural: bool = False):
        """``stream``: a cudaStream_t handle (int, e.g. ``torch.cuda.current_stream().cuda_stream``)
        to enqueue on instead of a library-owned stream.  ``allocator``: a pair of callables
        ``(alloc(nbytes) -> device pointer int, free(pointer))`` (e.g. torch's caching
        allocator) used for every buffer the library holds."""
        L = lib()
        self._rules = (Rule * max(1, len(cfg.rules)))()
        for q, r in enumerate(cfg.rules):
            self._rules[q] = Rule(r.src[0], r.src[1], r.dst[0], r.dst[1], r.kind, r.k,
                                  1 if r.plastic else 0, getattr(r, "delay_min", 0),
                                  getattr(r, "delay_max", 0), float(r.p))
        self._params = (C.c_double * max(1, len(cfg.params)))(*cfg.params)
        self._nccl = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        flags = (FLAG_EXTERNAL_EXCHANGE if external_exchange else 0) | \
                (FLAG_GLOBAL_ATOMICS if global_atomics else 0) | (FLAG_UNFUSED if unfused else 0) | \
                (FLAG_USER_STREAM if stream is not None else 0) | (FLAG_PROCEDURAL if procedural else 0)
        self._alloc_cbs = None
        if allocator is not None:
            alloc_fn, free_fn = allocator
            self._alloc_cbs = (DEV_ALLOC(lambda nbytes, ctx: alloc_fn(nbytes) or None),
                               DEV_FREE(lambda ptr, ctx: free_fn(ptr)))
        c = Config(ABI_VERSION, cfg.model, cfg.n, cfg.n_exc, self._rules, len(cfg.rules),
                   cfg.delay, cfg.dt_ms, cfg.seed, cfg.activity, self._params, len(cfg.params),
                   rank, world_size, slice_width, device,
                   C.cast(self._nccl, C.c_void_p) if self._nccl else None,
                   record_steps, flags, tile_width, ctas_per_tile, exchange,
                   stream if stream is not None else None,
                   C.cast(self._alloc_cbs[0], C.c_void_p) if self._alloc_cbs else None,
                   C.cast(self._alloc_cbs[1], C.c_void_p) if self._alloc_cbs else None, None)
        h = C.c_void_p()
        _check(L.spice_create_network(C.byref(c), C.byref(h)))
        self.h = h
        self.cfg, self.rank, self.world_size = cfg, rank, world_size
        self.n = cfg.n
        info = self.info()
        self.n_owned = info["n_owned"]
        self.slice_width = slice_width or default_slice_width(cfg.n, world_size)
        # u32 words of one rank's spike bitmap in the exchange buffers
        self.words_per_rank = (max(partition_owned_count(cfg.n, r, world_size, self.slice_width)
                                   for r in range(world_size)) + 31) // 32

    # lifecycle ---------------------------------------------------------------
    def free(self) -> None:
        if getattr(self, "h", None):
            lib().spice_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()

    # hot path ----------------------------------------------------------------
    def step(self, n_steps: int = 1) -> None:
        _check(lib().spice_step(self.h, n_steps))

    def read_spikes(self, t_begin: int, t_end: int):
        """List (per step) of ascending global spike IDs for steps [t_begin, t_end)."""
        L = lib()
        total = C.c_uint64(0)
        offs = np.zeros(t_end - t_begin + 1, dtype=np.uint64)
        st = L.spice_read_spikes(self.h, t_begin, t_end, None, 0, offs.ctypes.data, C.byref(total))
        if st not in (OK, ETRUNC):
            _check(st)
        ids = np.zeros(max(1, total.value), dtype=np.uint32)
        _check(L.spice_read_spikes(self.h, t_begin, t_end, ids.ctypes.data, ids.size,
                                   offs.ctypes.data, C.byref(total)))
        return [ids[int(offs[q]):int(offs[q + 1])].copy() for q in range(t_end - t_begin)]

    def read_spikes_into(self, t_begin: int, t_end: int, ids: np.ndarray, offs: np.ndarray) -> int:
        """Zero-allocation variant for timing loops; returns the spike count."""
        total = C.c_uint64(0)
        _check(lib().spice_read_spikes(self.h, t_begin, t_end, ids.ctypes.data, ids.size,
                                       offs.ctypes.data, C.byref(total)))
        return total.value

    def spikes_prefetch(self, t_begin: int, t_end: int, slot: int) -> None:
        """Enqueue the copy of steps [t_begin, t_end)'s spike bitmaps into pinned slot 0/1."""
        _check(lib().spice_spikes_prefetch(self.h, t_begin, t_end, slot))

    def spikes_collect_into(self, slot: int, ids: np.ndarray, offs: np.ndarray) -> int:
        """Wait for a prefetched slot and decode it (zero-allocation); returns the spike count."""
        total = C.c_uint64(0)
        _check(lib().spice_spikes_collect(self.h, slot, ids.ctypes.data, ids.size, offs.ctypes.data,
                                          C.byref(total)))
        return total.value

    # parity hooks --------------------------------------------------------------
    def connectivity(self, row_begin: int = 0, row_end: Optional[int] = None):
        L = lib()
        row_end = self.n if row_end is None else row_end
        total = C.c_uint64(0)
        offs = np.zeros(row_end - row_begin + 1, dtype=np.uint64)
        st = L.spice_read_connectivity(self.h, row_begin, row_end, None, 0, offs.ctypes.data, C.byref(total))
        if st not in (OK, ETRUNC):
            _check(st)
        tg = np.zeros(max(1, total.value), dtype=np.uint32)
        _check(L.spice_read_connectivity(self.h, row_begin, row_end, tg.ctypes.data, tg.size,
                                         offs.ctypes.data, C.byref(total)))
        return offs, tg[: total.value]

    def weights(self, row_begin: int = 0, row_end: Optional[int] = None) -> np.ndarray:
        """Plastic weights in the order of :meth:`connectivity` (static synapses read 0)."""
        L = lib()
        row_end = self.n if row_end is None else row_end
        total = C.c_uint64(0)
        st = L.spice_read_weights(self.h, row_begin, row_end, None, 0, C.byref(total))
        if st not in (OK, ETRUNC):
            _check(st)
        w = np.zeros(max(1, total.value), dtype=np.float32)
        _check(L.spice_read_weights(self.h, row_begin, row_end, w.ctypes.data, w.size, C.byref(total)))
        return w[: total.value]

    def delays(self, row_begin: int = 0, row_end: Optional[int] = None) -> np.ndarray:
        """Per-synapse delays (steps) in the order of :meth:`connectivity`."""
        L = lib()
        row_end = self.n if row_end is None else row_end
        total = C.c_uint64(0)
        st = L.spice_read_delays(self.h, row_begin, row_end, None, 0, C.byref(total))
        if st not in (OK, ETRUNC):
            _check(st)
        d = np.zeros(max(1, total.value), dtype=np.uint8)
        _check(L.spice_read_delays(self.h, row_begin, row_end, d.ctypes.data, d.size, C.byref(total)))
        return d[: total.value]

    def state(self, field: int) -> np.ndarray:
        dt = np.uint32 if field in (FIELD_REF, FIELD_ACC) else np.float32
        out = np.zeros(self.n_owned, dtype=dt)
        _check(lib().spice_read_state(self.h, field, out.ctypes.data, self.n_owned))
        return out

    def write_state(self, field: int, values) -> None:
        dt = np.uint32 if field in (FIELD_REF, FIELD_ACC) else np.float32
        a = np.ascontiguousarray(values, dtype=dt)
        _check(lib().spice_write_state(self.h, field, a.ctypes.data, a.size))

    def input(self, rel: int = 0):
        c = np.zeros(self.n_owned, dtype=np.uint32)
        p = np.zeros(self.n_owned, dtype=np.int64)
        _check(lib().spice_read_input(self.h, rel, c.ctypes.data, p.ctypes.data, self.n_owned))
        return c, p

    def force_next(self, ids: Sequence[int], mode: str = "replace") -> None:
        a = np.ascontiguousarray(ids, dtype=np.uint32)
        _check(lib().spice_force_spikes(self.h, a.ctypes.data, a.size, {"replace": 1, "add": 2}[mode]))

    def stats(self):
        s, f, d = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().spice_stats(self.h, C.byref(s), C.byref(f), C.byref(d)))
        return {"steps": s.value, "fired": f.value, "delivered": d.value}

    def info(self):
        o, s, nt, tw, c, b = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        _check(lib().spice_info(self.h, C.byref(o), C.byref(s), C.byref(nt), C.byref(tw), C.byref(c), C.byref(b)))
        return {"n_owned": o.value, "n_synapses": s.value, "n_tiles": nt.value, "tile_width": tw.value,
                "ctas_per_tile": c.value, "device_bytes": b.value}

    def setup_times(self):
        """Generator device ms and spice_create_network host wall ms of this slice."""
        g, w = C.c_double(), C.c_double()
        _check(lib().spice_setup_times(self.h, C.byref(g), C.byref(w)))
        return {"gen_ms": g.value, "create_ms": w.value}

    def profile(self, n_steps: int):
        """Average device ms per launch, each kernel bracketed by CUDA events on the
        library stream: update, deliver (unfused kernels), fused deliver(t)+update(t+1)
        (G = 1), exchange (all-gather + bitmap->list, G > 1).  Advances the network by
        2 * n_steps + 1 steps (G = 1) or n_steps steps."""
        out = np.zeros(5, dtype=np.float64)
        nk = C.c_uint32()
        _check(lib().spice_profile(self.h, n_steps, out.ctypes.data, 5, C.byref(nk)))
        return {"update": out[0], "deliver": out[1], "fused": out[2], "exchange": out[3],
                "fused_in_graph": out[4]}

    def debug_phases(self) -> np.ndarray:
        """SPICE_PHASES=1 diagnostics: (CTAs, 16) accumulated phase clocks (see spice.h)."""
        n = C.c_uint64()
        st = lib().spice_debug_phases(self.h, None, 0, C.byref(n))
        if st not in (OK, ETRUNC):
            _check(st)
        out = np.zeros(max(1, n.value), dtype=np.uint64)
        if n.value:
            _check(lib().spice_debug_phases(self.h, out.ctypes.data, out.size, C.byref(n)))
        return out[: n.value].reshape(-1, 16)

    def kernels_per_step(self) -> int:
        return lib().spice_kernels_per_step(self.h)

    def launches(self, n_steps: int) -> int:
        """Kernel launches spice_step(n_steps) enqueues (NCCL's own excluded)."""
        return lib().spice_launches(self.h, n_steps)

    @property
    def stream(self) -> int:
        return lib().spice_stream(self.h) or 0

    def sync(self) -> None:
        _check(lib().spice_sync(self.h))

    # external exchange (virtual ranks on one GPU) -------------------------------
    def exchange_begin(self) -> None:
        _check(lib().spice_exchange_begin(self.h))

    def exchange_end(self) -> None:
        _check(lib().spice_exchange_end(self.h))

    def exchange_end_fused(self) -> None:
        """G > 1 graph sequence: bitmap->list(t) + fused deliver(t)/update(t+1)."""
        _check(lib().spice_exchange_end_fused(self.h))

    def exchange_put_from(self, src: "Network") -> None:
        _check(lib().spice_exchange_put(self.h, src.h))

    def exchange_get_send(self, out, on_device: bool = False):
        """This rank's send bitmap -> `out` (numpy uint32[words_per_rank], or a device
        pointer / torch tensor with on_device=True)."""
        _check(lib().spice_exchange_get_send(self.h, _ptr(out), 1 if on_device else 0))
        return out

    def exchange_set_recv(self, rank: int, words, on_device: bool = False) -> None:
        """Fill rank `rank`'s receive segment from `words` (host array or device pointer)."""
        _check(lib().spice_exchange_set_recv(self.h, rank, _ptr(words), 1 if on_device else 0))

    # PEER exchange (device-initiated bitmap stores into every rank's window) --------
    def peer_handle(self) -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().spice_peer_handle(self.h, buf))
        return buf.raw

    def peer_connect(self, handles: Sequence[bytes]) -> None:
        """handles: the G ranks' peer_handle() bytes in rank order."""
        blob = b"".join(handles)
        assert len(blob) == 128 * self.world_size
        buf = C.create_string_buffer(blob, len(blob))
        _check(lib().spice_peer_connect(self.h, buf))
