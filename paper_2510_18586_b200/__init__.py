"""B200-native Tokencake Time-Scheduler hot path (arXiv 2510.18586): paged KV-block offload / predictive upload.

Thin ctypes binding over the C ABI in ``include/tokencake.h`` (``libtokencake.so``, built in-tree by
``paper_2510_18586_b200/build.py``).  Argument marshalling only: every step of the path — admission, allocation,
the gather/scatter kernels, the fused block-table remap, completion — runs in the library.  PyTorch is used only to
own device memory (the KV pool and block table tensors) and to name streams.

There is no fallback: if the shared library is missing or fails to load, importing this package raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtokencake.so")

OK, E_INVAL, E_NOBLOCKS, E_NOHOST, E_HANDLE, E_BUSY, E_CUDA, E_OOM, E_NODEV = 0, -1, -2, -3, -4, -5, -6, -7, -8
FP16, BF16 = 0, 1
XFER_AUTO, XFER_DIRECT, XFER_STAGED, XFER_COPY = 0, 1, 2, 3
DTYPES = {"fp16": FP16, "bf16": BF16}

SYMBOLS = [
    "tc_pool_desc_init", "tc_pool_create", "tc_pool_create_ex", "tc_pool_destroy", "tc_pool_kv",
    "tc_set_compute_stream", "tc_streams", "tc_set_xfer_mode", "tc_calibrate", "tc_set_launch_config", "tc_fill_kv", "tc_partition_reserve",
    "tc_agent_add", "tc_alloc", "tc_agent_free", "tc_offload", "tc_upload", "tc_offload_batch", "tc_upload_batch",
    "tc_cycle", "tc_reserve_begin", "tc_reserve_tick", "tc_reserve_cancel", "tc_reserve_info",
    "tc_query", "tc_wait", "tc_stream_wait", "tc_sync", "tc_retire", "tc_retire_lag", "tc_block_table", "tc_block_table_dev", "tc_handle_info",
    "tc_handle_host", "tc_handle_read", "tc_stats", "tc_timing", "tc_timeline", "tc_trace", "tc_trace_read", "tc_strerror", "tc_last_error", "tc_gather_dev",
    "tc_scatter_dev",
    # decision layers (paper_2510_18586_b200/sched.py binds them)
    "tc_fc_predict", "tc_fc_observe", "tc_transfer_ms", "tc_xfer_model_measure", "tc_should_offload",
    "tc_plan_upload", "tc_static_priority", "tc_dynamic_priority", "tc_select_critical", "tc_update_reservations",
    "tc_apply_reservations", "tc_ts_params_init", "tc_ts_create", "tc_ts_destroy", "tc_ts_call_start", "tc_ts_tick",
    "tc_ts_call_finish", "tc_ts_forecast", "tc_ss_params_init", "tc_ss_create", "tc_ss_destroy", "tc_ss_update",
    "tc_ss_critical_inversion",
]


class TcError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"tokencake status {status}: {msg}")
        self.status = status


class PoolDesc(ctypes.Structure):
    _fields_ = [
        ("layers", ctypes.c_int32), ("kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
        ("block_tokens", ctypes.c_int32), ("dtype", ctypes.c_int32), ("n_blocks", ctypes.c_int64),
        ("device", ctypes.c_int32), ("shard_rank", ctypes.c_int32), ("shard_world", ctypes.c_int32),
        ("host_slots", ctypes.c_int64), ("n_classes", ctypes.c_int32), ("max_agents", ctypes.c_int32),
        ("max_blocks_per_agent", ctypes.c_int32), ("kv_dev", ctypes.c_void_p), ("table_dev", ctypes.c_void_p),
        ("xfer_d2h", ctypes.c_int32), ("xfer_h2d", ctypes.c_int32), ("staging_bytes", ctypes.c_int64),
        ("desc_bytes", ctypes.c_int64), ("unbuffered", ctypes.c_int32), ("peer_device", ctypes.c_int32),
        ("peer_slots", ctypes.c_int64),
    ]


class Timing(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 9), ("count", ctypes.c_int64 * 9), ("bytes", ctypes.c_int64 * 9),
                ("kernel_ms", ctypes.c_double * 9), ("kernel_count", ctypes.c_int64 * 9),
                ("kernel_bytes", ctypes.c_int64 * 9)]


class Calibration(ctypes.Structure):
    _fields_ = [("d2h", ctypes.c_int32), ("h2d", ctypes.c_int32), ("probe_bytes", ctypes.c_int64),
                ("gbs", ctypes.c_double * 4), ("direct_max_bytes", ctypes.c_int64 * 2)]


class TraceRec(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("agent", ctypes.c_int32), ("handle", ctypes.c_uint64),
                ("blocks", ctypes.c_int64), ("bytes", ctypes.c_int64), ("t_call_ns", ctypes.c_int64),
                ("t_enqueued_ns", ctypes.c_int64), ("t_done_ns", ctypes.c_int64)]


class Span(ctypes.Structure):
    _fields_ = [("sync", ctypes.c_int64), ("kind", ctypes.c_int32), ("start_ms", ctypes.c_double),
                ("end_ms", ctypes.c_double), ("bytes", ctypes.c_int64)]


TIMING_KINDS = ("offload_kernel", "upload_kernel", "device_kernel", "memcpy_d2h", "memcpy_h2d", "offload_peer_kernel",
                "upload_peer_kernel", "offload_direct_kernel", "upload_direct_kernel")
KERNEL_KINDS = (0, 1, 2, 5, 6, 7, 8)


class Stats(ctypes.Structure):
    _fields_ = [
        ("n_blocks", ctypes.c_int64), ("free_blocks", ctypes.c_int64), ("alloc_blocks", ctypes.c_int64),
        ("pending_blocks", ctypes.c_int64), ("host_slots", ctypes.c_int64), ("host_free", ctypes.c_int64),
        ("host_used", ctypes.c_int64), ("host_released", ctypes.c_int64), ("chunk_bytes", ctypes.c_int64),
        ("block_bytes", ctypes.c_int64), ("n_classes", ctypes.c_int32), ("n_agents", ctypes.c_int32),
        ("reserved", ctypes.c_int64 * 64), ("claimed", ctypes.c_int64 * 64), ("live_handles", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64), ("memcpy_calls", ctypes.c_int64), ("bytes_d2h", ctypes.c_int64),
        ("bytes_h2d", ctypes.c_int64), ("xfer_d2h", ctypes.c_int32), ("xfer_h2d", ctypes.c_int32),
        ("reserved_blocks", ctypes.c_int64), ("peer_slots", ctypes.c_int64), ("peer_free", ctypes.c_int64),
        ("peer_used", ctypes.c_int64),
    ]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH) or _build.stale():
        _build.build()
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U64, VP = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
    PI32, PI64, PU64 = ctypes.POINTER(I32), ctypes.POINTER(I64), ctypes.POINTER(U64)
    sig = {
        "tc_pool_desc_init": (None, [ctypes.POINTER(PoolDesc), I32, I32, I32, I32, I32, I64]),
        "tc_pool_create": (I32, [I32, I32, I32, I32, I32, I64, ctypes.POINTER(P)]),
        "tc_pool_create_ex": (I32, [ctypes.POINTER(PoolDesc), ctypes.POINTER(P)]),
        "tc_pool_destroy": (None, [P]),
        "tc_pool_kv": (I32, [P, ctypes.POINTER(VP), PI64]),
        "tc_set_compute_stream": (I32, [P, VP]),
        "tc_streams": (I32, [P, ctypes.POINTER(VP), ctypes.POINTER(VP)]),
        "tc_set_xfer_mode": (I32, [P, I32, I32]),
        "tc_calibrate": (I32, [P, I64, ctypes.POINTER(Calibration)]),
        "tc_set_launch_config": (I32, [P, I32, I32, I32, I32]),
        "tc_fill_kv": (I32, [P, U64]),
        "tc_partition_reserve": (I32, [P, I32, I64]),
        "tc_agent_add": (I32, [P, I32, I32]),
        "tc_alloc": (I32, [P, I32, I64, PI32]),
        "tc_agent_free": (I32, [P, I32]),
        "tc_offload": (I32, [P, I32, PI32, I64, PU64]),
        "tc_upload": (I32, [P, U64, PI32]),
        "tc_offload_batch": (I32, [P, I32, PI32, PI64, PI32, PU64]),
        "tc_upload_batch": (I32, [P, I32, PU64, PI64, PI32]),
        "tc_cycle": (I32, [P, I32, PU64, PI64, PI32, I32, PI32, PI64, PI32, PU64]),
        "tc_reserve_begin": (I32, [P, U64, I32]),
        "tc_reserve_tick": (I32, [P]),
        "tc_reserve_cancel": (I32, [P, U64]),
        "tc_reserve_info": (I32, [P, U64, PI64, PI64]),
        "tc_query": (I32, [P, U64]),
        "tc_wait": (I32, [P, U64]),
        "tc_stream_wait": (I32, [P, U64, VP]),
        "tc_sync": (I32, [P]),
        "tc_retire": (I32, [P]),
        "tc_retire_lag": (I32, [P, I32]),
        "tc_block_table": (I32, [P, I32, PI32, I64, PI64]),
        "tc_block_table_dev": (I32, [P, ctypes.POINTER(PI32), PI64]),
        "tc_handle_info": (I32, [P, U64, PI32, PI64, PI32]),
        "tc_handle_host": (I32, [P, U64, I64, ctypes.POINTER(VP)]),
        "tc_handle_read": (I32, [P, U64, I64, VP, PI32]),
        "tc_stats": (I32, [P, ctypes.POINTER(Stats)]),
        "tc_timing": (I32, [P, I32, ctypes.POINTER(Timing)]),
        "tc_timeline": (I32, [P, I64, ctypes.POINTER(Span), PI64]),
        "tc_trace": (I32, [P, I64]),
        "tc_trace_read": (I32, [P, ctypes.POINTER(TraceRec), I64, PI64]),
        "tc_strerror": (ctypes.c_char_p, [I32]),
        "tc_last_error": (ctypes.c_char_p, [P]),
        "tc_gather_dev": (I32, [P, PI32, I64, VP, VP]),
        "tc_scatter_dev": (I32, [P, VP, PI32, I64, VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class Pool:
    """One paged KV pool on one CUDA device (or metadata-only with ``device=-1``), driven through the C ABI.

    Method vocabulary (shared with the test replayer): reserve, agent_add, alloc, offload, upload, offload_batch,
    upload_batch, sync, agent_free, block_table, stats, plus query / wait / stream_wait and device-tier helpers.
    """

    def __init__(self, layers: int, kv_heads: int, head_dim: int, block_tokens: int = 16, dtype: str = "bf16",
                 n_blocks: int = 64, *, device: int = 0, shard_rank: int = 0, shard_world: int = 1,
                 host_slots: int = 0, n_classes: int = 8, max_agents: int = 1024, max_blocks_per_agent: int = 4096,
                 xfer_d2h: int = XFER_AUTO, xfer_h2d: int = XFER_AUTO, staging_bytes: int = 0,
                 torch_memory: bool = True, unbuffered: bool = False, peer_device: int = -1, peer_slots: int = 0):
        d = PoolDesc()
        lib.tc_pool_desc_init(ctypes.byref(d), layers, kv_heads, head_dim, block_tokens, DTYPES[dtype], n_blocks)
        d.device = device
        d.shard_rank, d.shard_world = shard_rank, shard_world
        d.host_slots = host_slots
        d.n_classes, d.max_agents, d.max_blocks_per_agent = n_classes, max_agents, max_blocks_per_agent
        d.xfer_d2h, d.xfer_h2d = xfer_d2h, xfer_h2d
        d.staging_bytes = staging_bytes
        d.unbuffered = 1 if unbuffered else 0
        d.peer_device, d.peer_slots = peer_device, peer_slots
        self._keep = []
        self.device = device
        self.meta_only = device < 0
        if not self.meta_only and torch_memory:
            import torch   # device memory is owned by PyTorch (plumbing), the pointers are handed to the library
            hl = kv_heads // shard_world
            kv_bytes = layers * 2 * n_blocks * block_tokens * hl * head_dim * 2
            kv = torch.empty(kv_bytes, dtype=torch.uint8, device=f"cuda:{device}")
            tab = torch.empty(max_agents * max_blocks_per_agent, dtype=torch.int32, device=f"cuda:{device}")
            torch.cuda.synchronize(device)
            d.kv_dev, d.table_dev = kv.data_ptr(), tab.data_ptr()
            self._keep = [kv, tab]
        h = ctypes.c_void_p()
        self._check(lib.tc_pool_create_ex(ctypes.byref(d), ctypes.byref(h)), None)
        self._h = h
        self.desc = d
        s = self.stats()
        self.chunk_bytes, self.block_bytes = s["chunk_bytes"], s["block_bytes"]
        self.L, self.H, self.D, self.T = layers, kv_heads, head_dim, block_tokens
        self.Hl = kv_heads // shard_world
        self.N = n_blocks
        self.max_bpa = max_blocks_per_agent

    # ------------------------------------------------------------------ plumbing
    def _check(self, st: int, h=None):
        if st != OK:
            msg = lib.tc_strerror(st).decode()
            if h is not None or getattr(self, "_h", None) is not None:
                le = lib.tc_last_error(h if h is not None else self._h)
                if le:
                    msg += f" ({le.decode()})"
            raise TcError(st, msg)

    def close(self):
        if getattr(self, "_h", None):
            lib.tc_pool_destroy(self._h)
            self._h = None
        if self._keep:
            self._keep = []
            import torch   # hand the pool's HBM back (the caching allocator would keep tens of GiB reserved)
            torch.cuda.empty_cache()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # ------------------------------------------------------------------ vocabulary
    def reserve(self, cls: int, n: int):
        self._check(lib.tc_partition_reserve(self._h, cls, n))

    def agent_add(self, agent: int, cls: int):
        self._check(lib.tc_agent_add(self._h, agent, cls))

    def alloc(self, agent: int, n: int) -> list:
        out = np.empty(max(n, 1), dtype=np.int32)
        self._check(lib.tc_alloc(self._h, agent, n, _ptr(out, ctypes.c_int32)))
        return out[:n].tolist()

    def agent_free(self, agent: int):
        self._check(lib.tc_agent_free(self._h, agent))

    def offload(self, agent: int, ids) -> int:
        a = _i32(ids)
        h = ctypes.c_uint64()
        self._check(lib.tc_offload(self._h, agent, _ptr(a, ctypes.c_int32), a.size, ctypes.byref(h)))
        return h.value

    def upload(self, h: int) -> list:
        agent, n, state = self.handle_info(h) if h else (0, 1, 0)
        out = np.empty(max(n, 1), dtype=np.int32)
        self._check(lib.tc_upload(self._h, h, _ptr(out, ctypes.c_int32)))
        return out[:n].tolist()

    def offload_batch(self, items) -> list:
        agents = _i32([a for a, _ in items])
        offs = np.zeros(len(items) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(ids) for _, ids in items])
        ids = _i32([b for _, x in items for b in x]) if offs[-1] else np.zeros(1, np.int32)
        out = np.zeros(max(len(items), 1), dtype=np.uint64)
        self._check(lib.tc_offload_batch(self._h, len(items), _ptr(agents, ctypes.c_int32),
                                         _ptr(offs, ctypes.c_int64), _ptr(ids, ctypes.c_int32),
                                         _ptr(out, ctypes.c_uint64)))
        return [int(x) for x in out[:len(items)]]

    def offload_batch_arrays(self, agents: np.ndarray, offsets: np.ndarray, ids: np.ndarray) -> np.ndarray:
        """Zero-copy batch entry for prebuilt int32/int64 arrays (bench hot loop)."""
        out = np.zeros(len(agents), dtype=np.uint64)
        self._check(lib.tc_offload_batch(self._h, len(agents), _ptr(agents, ctypes.c_int32),
                                         _ptr(offsets, ctypes.c_int64), _ptr(ids, ctypes.c_int32),
                                         _ptr(out, ctypes.c_uint64)))
        return out

    def upload_batch(self, hs) -> list:
        hs_a = np.ascontiguousarray(np.asarray(hs, dtype=np.uint64))
        sizes = []
        for h in hs:
            try:
                sizes.append(self.handle_info(int(h))[1])
            except TcError:
                sizes.append(0)
        offs = np.zeros(len(hs) + 1, dtype=np.int64)
        offs[1:] = np.cumsum(sizes)
        out = np.empty(max(int(offs[-1]), 1), dtype=np.int32)
        self._check(lib.tc_upload_batch(self._h, len(hs), _ptr(hs_a, ctypes.c_uint64), _ptr(offs, ctypes.c_int64),
                                        _ptr(out, ctypes.c_int32)))
        return [out[offs[k]:offs[k + 1]].tolist() for k in range(len(hs))]

    def upload_batch_arrays(self, hs: np.ndarray, offsets: np.ndarray, out: np.ndarray) -> np.ndarray:
        self._check(lib.tc_upload_batch(self._h, len(hs), _ptr(hs, ctypes.c_uint64), _ptr(offsets, ctypes.c_int64),
                                        _ptr(out, ctypes.c_int32)))
        return out

    def sync(self):
        self._check(lib.tc_sync(self._h))

    def retire(self, lag: int = 1):
        """tc_retire: retire what was enqueued before the previous retire / sync point, without draining;
        lag > 1 (tc_retire_lag): before the lag-th previous point."""
        self._check(lib.tc_retire(self._h) if lag == 1 else lib.tc_retire_lag(self._h, int(lag)))

    def cycle(self, up_handles, off_items):
        """One scheduling cycle (tc_cycle): uploads of `up_handles`, then offloads [(agent, ids), ...].
        Returns (new id lists per upload handle, new handles per offload item)."""
        hs = np.ascontiguousarray(np.asarray(up_handles, dtype=np.uint64).reshape(-1))
        sizes = []
        for h in hs:
            try:
                sizes.append(self.handle_info(int(h))[1])
            except TcError:
                sizes.append(0)
        uoff = np.zeros(len(hs) + 1, dtype=np.int64)
        uoff[1:] = np.cumsum(sizes)
        agents = _i32([a for a, _ in off_items])
        ooff = np.zeros(len(off_items) + 1, dtype=np.int64)
        ooff[1:] = np.cumsum([len(x) for _, x in off_items])
        ids = _i32([b for _, x in off_items for b in x]) if ooff[-1] else np.zeros(1, np.int32)
        new, out_h = self.cycle_arrays(hs, uoff, agents, ooff, ids)
        return [new[uoff[k]:uoff[k + 1]].tolist() for k in range(len(hs))], [int(x) for x in out_h]

    def cycle_arrays(self, hs: np.ndarray, uoff: np.ndarray, agents: np.ndarray, ooff: np.ndarray,
                     ids: np.ndarray):
        """Zero-copy tc_cycle for prebuilt arrays (bench hot loop)."""
        new = np.empty(max(int(uoff[-1]), 1), dtype=np.int32)
        out_h = np.zeros(max(len(agents), 1), dtype=np.uint64)
        self._check(lib.tc_cycle(self._h, len(hs), _ptr(hs, ctypes.c_uint64), _ptr(uoff, ctypes.c_int64),
                                 _ptr(new, ctypes.c_int32), len(agents), _ptr(agents, ctypes.c_int32),
                                 _ptr(ooff, ctypes.c_int64), _ptr(ids, ctypes.c_int32),
                                 _ptr(out_h, ctypes.c_uint64)))
        return new[:int(uoff[-1])], out_h[:len(agents)]

    def reserve_begin(self, h: int, cycles: int):
        self._check(lib.tc_reserve_begin(self._h, h, cycles))

    def reserve_tick(self):
        self._check(lib.tc_reserve_tick(self._h))

    def reserve_cancel(self, h: int):
        self._check(lib.tc_reserve_cancel(self._h, h))

    def reserve_info(self, h: int):
        k, n = ctypes.c_int64(), ctypes.c_int64()
        self._check(lib.tc_reserve_info(self._h, h, ctypes.byref(k), ctypes.byref(n)))
        return k.value, n.value

    def query(self, h: int) -> bool:
        st = lib.tc_query(self._h, h)
        if st == E_BUSY:
            return False
        self._check(st)
        return True

    def wait(self, h: int):
        self._check(lib.tc_wait(self._h, h))

    def stream_wait(self, h: int, stream_ptr: int):
        self._check(lib.tc_stream_wait(self._h, h, stream_ptr))

    def block_table(self, agent: int) -> list:
        return self.block_table_np(agent).tolist()

    def block_table_np(self, agent: int) -> np.ndarray:
        """The agent's block table as an int32 array (-1 = on host): one tc_block_table call into a row-sized
        buffer (the hot-loop form)."""
        n = ctypes.c_int64()
        out = np.empty(self.max_bpa, dtype=np.int32)
        self._check(lib.tc_block_table(self._h, agent, _ptr(out, ctypes.c_int32), out.size, ctypes.byref(n)))
        return out[:n.value]

    def handle_info(self, h: int):
        a, n, s = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32()
        self._check(lib.tc_handle_info(self._h, h, ctypes.byref(a), ctypes.byref(n), ctypes.byref(s)))
        return a.value, n.value, s.value

    def handle_host_bytes(self, h: int, i: int) -> np.ndarray:
        """Copy of the offloaded image [L][2][C] of block i of a handle, from its host slot or peer-tier slot
        (tc_handle_read waits for the handle's transfer)."""
        buf = np.empty(self.block_bytes, dtype=np.uint8)
        tier = ctypes.c_int32()
        self._check(lib.tc_handle_read(self._h, h, i, buf.ctypes.data, ctypes.byref(tier)))
        return buf.reshape(self.L, 2, self.chunk_bytes)

    def handle_tier(self, h: int, i: int = 0) -> int:
        """0 = host tier, 1 = peer tier (NEXT-2) for block i of an offloaded handle."""
        buf = np.empty(self.block_bytes, dtype=np.uint8)
        tier = ctypes.c_int32()
        self._check(lib.tc_handle_read(self._h, h, i, buf.ctypes.data, ctypes.byref(tier)))
        return tier.value

    def stats(self) -> dict:
        s = Stats()
        self._check(lib.tc_stats(self._h, ctypes.byref(s)))
        d = {k: getattr(s, k) for k, _ in Stats._fields_ if k not in ("reserved", "claimed")}
        d["reserved"] = list(s.reserved[:s.n_classes])
        d["claimed"] = list(s.claimed[:s.n_classes])
        d["free"], d["alloc"], d["pending"] = s.free_blocks, s.alloc_blocks, s.pending_blocks
        return d

    def timing(self, enable: bool | int = True) -> dict:
        """Enable/disable per-launch timing; returns {kind: (ms, count, bytes)} accumulated since the last call:
        event spans per kind (TIMING_KINDS) plus device-side kernel durations under 'dev_<kind>'."""
        t = Timing()
        self._check(lib.tc_timing(self._h, int(enable), ctypes.byref(t)))
        out = {k: (t.ms[i], t.count[i], t.bytes[i]) for i, k in enumerate(TIMING_KINDS)}
        for i in KERNEL_KINDS:
            out["dev_" + TIMING_KINDS[i]] = (t.kernel_ms[i], t.kernel_count[i], t.kernel_bytes[i])
        return out

    def trace(self, cap: int = 100000):
        """Arm (cap > 0) or stop (0) the per-call trace (tc_trace)."""
        self._check(lib.tc_trace(self._h, cap))

    def trace_read(self, cap: int = 100000) -> list:
        """Per-call records since the last read: dicts with op ('offload' | 'upload'), agent, handle, blocks, bytes,
        t_call_ns, t_enqueued_ns, t_done_ns (host steady clock)."""
        buf = (TraceRec * cap)()
        n = ctypes.c_int64()
        self._check(lib.tc_trace_read(self._h, buf, cap, ctypes.byref(n)))
        ops = {1: "offload", 2: "upload"}
        return [{"op": ops[buf[i].op], **{k: getattr(buf[i], k) for k, _ in TraceRec._fields_ if k != "op"}}
                for i in range(n.value)]

    def timeline_arm(self, cap: int = 100000):
        n = ctypes.c_int64()
        self._check(lib.tc_timeline(self._h, cap, None, ctypes.byref(n)))

    def timeline(self, cap: int = 100000) -> list:
        """[(sync_index, kind_name, start_ms, end_ms, bytes), ...] recorded since timeline_arm()."""
        buf = (Span * cap)()
        n = ctypes.c_int64()
        self._check(lib.tc_timeline(self._h, cap, buf, ctypes.byref(n)))
        return [(buf[i].sync, TIMING_KINDS[buf[i].kind], buf[i].start_ms, buf[i].end_ms, buf[i].bytes)
                for i in range(n.value)]

    def streams(self):
        up, off = ctypes.c_void_p(), ctypes.c_void_p()
        self._check(lib.tc_streams(self._h, ctypes.byref(up), ctypes.byref(off)))
        return up.value, off.value

    def set_compute_stream(self, stream_ptr: int | None):
        self._check(lib.tc_set_compute_stream(self._h, stream_ptr))

    def set_xfer_mode(self, d2h: int, h2d: int):
        self._check(lib.tc_set_xfer_mode(self._h, d2h, h2d))

    def calibrate(self, probe_bytes: int = 256 << 20) -> dict:
        """tc_calibrate: time a concurrent offload + upload of probe_bytes for each {DIRECT, STAGED} combination and
        make AUTO directions take the fastest; returns the chosen modes and GB/s per combination."""
        c = Calibration()
        self._check(lib.tc_calibrate(self._h, probe_bytes, ctypes.byref(c)))
        names = {XFER_DIRECT: "direct", XFER_STAGED: "staged"}
        return {"d2h": names[c.d2h], "h2d": names[c.h2d], "probe_bytes": c.probe_bytes,
                "gbs": {f"{a}/{b}": c.gbs[2 * i + j] for i, a in enumerate(("direct", "staged"))
                        for j, b in enumerate(("direct", "staged"))},
                "direct_max_bytes": {"d2h": int(c.direct_max_bytes[0]), "h2d": int(c.direct_max_bytes[1])}}

    def set_launch_config(self, path: int, ctas: int = 0, threads: int = 256, variant: int = 0):
        """path 0 = direct D2H, 1 = direct H2D, 2 = device-side (staged/device tier); variant 1 = TMA bulk."""
        self._check(lib.tc_set_launch_config(self._h, path, ctas, threads, variant))

    def fill(self, seed: int):
        self._check(lib.tc_fill_kv(self._h, seed))

    def kv_ptr(self) -> int:
        p, c = ctypes.c_void_p(), ctypes.c_int64()
        self._check(lib.tc_pool_kv(self._h, ctypes.byref(p), ctypes.byref(c)))
        return p.value

    def kv_tensor(self):
        """The KV pool as a torch uint8 tensor view [L][2][N][C] (torch-owned memory)."""
        return self._keep[0].view(self.L, 2, self.N, self.chunk_bytes)

    def table_tensor(self):
        return self._keep[1].view(-1, self.max_bpa)

    def gather_dev(self, ids, dst_ptr: int, stream_ptr: int | None = None):
        a = _i32(ids)
        self._check(lib.tc_gather_dev(self._h, _ptr(a, ctypes.c_int32), a.size, dst_ptr, stream_ptr))

    def scatter_dev(self, src_ptr: int, ids, stream_ptr: int | None = None):
        a = _i32(ids)
        self._check(lib.tc_scatter_dev(self._h, src_ptr, _ptr(a, ctypes.c_int32), a.size, stream_ptr))
