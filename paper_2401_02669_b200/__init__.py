"""B200-native DistAttention decode path (Infinite-LLM, arXiv 2401.02669).

Python host mirror of the C ABI in ``include/dattn.h`` (ctypes, no torch types
in the boundary). The compute runs in ``_lib/libdattn.so`` (sm_100a kernels);
there is no CPU fallback. The library is mapped on first use (``lib``,
``Store``, ``comm_unique_id``, ...), so the pure host modules ``workloads`` and
``sharding`` import without it (bench.py's reference arm must not map the
product library); any GPU-path call without the built library raises
``ImportError``.

Reference interface mirrored: ``kvsched::attn`` (proj/include/kvsched/
distattention.hpp:16-95) and the C ABI conventions of proj/include/kvsched.h
(status codes, thread-local last error). Errors map onto the reference's two
exception kinds: ``ContractError`` (caller bug, common.hpp:11-15) and
``InputError`` (bad data, common.hpp:17-20).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DATTN_LIB") or os.path.join(_HERE, "_lib", "libdattn.so")  # DATTN_LIB: A/B builds

BF16, F32, F64 = 0, 1, 2
MEM_DEVICE, MEM_HOST = 0, 1
F_NO_OUTPUT, F_CHECK_FINITE = 1, 2
ELEM_BYTES = {BF16: 2, F32: 4, F64: 8}

OK, ERR_INVALID_ARGUMENT, ERR_INPUT, ERR_CONTRACT, ERR_INTERNAL, ERR_CUDA, ERR_NCCL, ERR_CAPACITY = range(8)


class DattnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[dattn status {status}] {msg}")
        self.status = status


class ContractError(DattnError):
    """Precondition violated (kvsched::ContractError, common.hpp:11-15)."""


class InputError(DattnError):
    """Rejected data (kvsched::InputError, common.hpp:17-20)."""


class CapacityError(DattnError):
    """Page pool / block table exhausted (RManager::alloc_local returning false)."""


class StoreConfig(ctypes.Structure):
    _fields_ = [
        ("head_dim", ctypes.c_int), ("num_q_heads", ctypes.c_int), ("num_kv_heads", ctypes.c_int),
        ("scale", ctypes.c_double), ("dtype", ctypes.c_int), ("page_tokens", ctypes.c_int),
        ("num_pages", ctypes.c_int64), ("max_seqs", ctypes.c_int),
        ("max_pages_per_seq", ctypes.c_int), ("device", ctypes.c_int),
    ]


class StoreInfo(ctypes.Structure):
    _fields_ = [
        ("padded_dim", ctypes.c_int), ("elem_bytes", ctypes.c_int), ("record_elems", ctypes.c_int),
        ("record_bytes", ctypes.c_int), ("free_pages", ctypes.c_int64),
        ("used_pages", ctypes.c_int64), ("pool_bytes", ctypes.c_int64), ("num_sms", ctypes.c_int),
    ]


class Range(ctypes.Structure):
    """One rBlock: tokens [tok_begin, tok_end) of a block-table row, feeding
    output row ``out_row`` (kv_head -1: every kv head)."""
    _fields_ = [
        ("seq", ctypes.c_int32), ("out_row", ctypes.c_int32), ("kv_head", ctypes.c_int32),
        ("reserved", ctypes.c_int32), ("tok_begin", ctypes.c_int64), ("tok_end", ctypes.c_int64),
    ]

    def __init__(self, seq=0, out_row=0, tok_begin=0, tok_end=0, kv_head=-1):
        super().__init__(seq, out_row, kv_head, 0, tok_begin, tok_end)


class Batch(ctypes.Structure):
    _fields_ = [
        ("num_rows", ctypes.c_int32), ("num_ranges", ctypes.c_int32),
        ("ranges", ctypes.POINTER(Range)), ("chunk_tokens", ctypes.c_int32),
        ("flags", ctypes.c_int32), ("scale", ctypes.c_double),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("ma_launches", ctypes.c_int64), ("merge_launches", ctypes.c_int64),
        ("ma_timed", ctypes.c_int64), ("merge_timed", ctypes.c_int64),
        ("ma_ms", ctypes.c_double), ("merge_ms", ctypes.c_double),
        ("last_items", ctypes.c_int64), ("last_chunks", ctypes.c_int64),
        ("last_plan_bytes", ctypes.c_int64), ("last_chunk_tokens", ctypes.c_int32),
        ("ma_grid", ctypes.c_int32), ("last_kernel", ctypes.c_int32), ("last_exchange", ctypes.c_int32),
        ("comm_timed", ctypes.c_int64), ("comm_ms", ctypes.c_double),
    ]


class MergeDesc(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int32), ("heads", ctypes.c_int32), ("row_begin", ctypes.c_void_p),
        ("n_uniform", ctypes.c_int32), ("row_mul", ctypes.c_int64), ("c_stride", ctypes.c_int64),
    ]


_FUNCS = {
    "dattn_last_error": (ctypes.c_char_p, []),
    "dattn_string_free": (None, [ctypes.c_void_p]),
    "dattn_abi_version": (ctypes.c_int, []),
    "dattn_launch_count": (ctypes.c_int64, [ctypes.c_int]),
    "dattn_store_create": (ctypes.c_int, [ctypes.POINTER(StoreConfig), ctypes.POINTER(ctypes.c_void_p)]),
    "dattn_store_destroy": (None, [ctypes.c_void_p]),
    "dattn_store_get_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(StoreInfo)]),
    "dattn_store_set_timing": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "dattn_store_get_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(Stats)]),
    "dattn_store_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "dattn_store_set_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "dattn_store_synchronize": (ctypes.c_int, [ctypes.c_void_p]),
    "dattn_seq_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int32)]),
    "dattn_seq_resize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64]),
    "dattn_seq_release": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]),
    "dattn_seq_tokens": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]),
    "dattn_seq_block_table": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                             ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
    "dattn_kv_write": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.c_int]),
    "dattn_kv_read": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "dattn_kv_append": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int]),
    "dattn_kv_synthetic_rows": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_uint64, ctypes.c_float, ctypes.c_float, ctypes.c_void_p,
                                               ctypes.c_void_p]),
    "dattn_kv_fill_synthetic": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64,
                                               ctypes.c_uint32, ctypes.c_int64, ctypes.c_float,
                                               ctypes.c_float]),
    "dattn_q_fill_synthetic": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                              ctypes.c_uint64, ctypes.c_uint32, ctypes.c_float]),
    "dattn_decode": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Batch), ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "dattn_micro_attention": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Batch), ctypes.c_void_p,
                                             ctypes.c_void_p]),
    "dattn_merge_partials": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(MergeDesc), ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p]),
    "dattn_comm_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "dattn_comm_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
    "dattn_comm_abort": (ctypes.c_int, [ctypes.c_void_p]),
    "dattn_comm_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_int)]),
    "dattn_decode_sharded": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Batch), ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_int]),
    "dattn_kv_send": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]),
    "dattn_kv_recv": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]),
    "dattn_kv_pull": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_int64]),
    "dattn_kv_migration_join": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "dattn_ledger_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_void_p)]),
    "dattn_ledger_destroy": (None, [ctypes.c_void_p]),
    "dattn_ledger_admit": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_int)]),
    "dattn_ledger_ensure_slot": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    "dattn_ledger_advance": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64]),
    "dattn_ledger_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.c_void_p]),
    "dattn_ledger_release": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
    "dattn_ledger_instance": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "dattn_ledger_request": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "dattn_ledger_blocks": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]),
    "dattn_ledger_segments": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "dattn_ledger_borrowed": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "dattn_verify_attention": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                                              ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int)]),
    "dattn_host_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "dattn_host_free": (None, [ctypes.c_void_p]),
    "dattn_device_alloc": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "dattn_device_free": (None, [ctypes.c_void_p, ctypes.c_void_p]),
    "dattn_memcpy": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                    ctypes.c_int]),
}

EXPORTED_SYMBOLS = tuple(_FUNCS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA library is not built (run __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_LOCAL)
    for name, (res, args) in _FUNCS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _LazyLib:
    """ctypes handle of libdattn.so, loaded on first attribute access."""
    _h = None

    def __getattr__(self, name):
        if _LazyLib._h is None:
            _LazyLib._h = _load()
        return getattr(_LazyLib._h, name)

    @staticmethod
    def loaded() -> bool:
        return _LazyLib._h is not None


lib = _LazyLib()


def last_error() -> str:
    s = lib.dattn_last_error()
    return s.decode() if s else ""


def check(status: int) -> None:
    if status == OK:
        return
    msg = last_error()
    if status == ERR_CONTRACT:
        raise ContractError(status, msg)
    if status == ERR_INPUT:
        raise InputError(status, msg)
    if status == ERR_CAPACITY:
        raise CapacityError(status, msg)
    raise DattnError(status, msg)


def ptr(x) -> Optional[int]:
    """Raw address of a torch tensor / numpy array / int (None stays None)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)!r}")


def launch_count(reset: bool = False) -> int:
    return int(lib.dattn_launch_count(1 if reset else 0))


def blocks_for_tokens(tokens: int, block_size_tokens: int) -> int:
    """perfmodel.cpp:178-182 -- the page-count contract of the block ledger."""
    return (tokens + block_size_tokens - 1) // block_size_tokens


def gqa_kv_head(query_head: int, num_q_heads: int, num_kv_heads: int) -> int:
    """distattention.cpp:176-181 -- contiguous query-head groups."""
    if num_q_heads < 1 or num_kv_heads < 1 or num_q_heads % num_kv_heads:
        raise ContractError(ERR_CONTRACT, "num_q_heads must be a multiple of num_kv_heads")
    if not 0 <= query_head < num_q_heads:
        raise ContractError(ERR_CONTRACT, "query_head out of range")
    return query_head // (num_q_heads // num_kv_heads)


def effective_scale(head_dim: int, scale: float = 0.0) -> float:
    """distattention.cpp:35-37."""
    return scale if scale > 0.0 else 1.0 / math.sqrt(head_dim)


def padded_dim(head_dim: int) -> int:
    for dp in (16, 32, 64, 128, 256, 512):
        if head_dim <= dp:
            return dp
    raise ContractError(ERR_CONTRACT, "head_dim must be <= 512")


class RangeArray:
    """Ranges packed once into a ctypes array; decode calls accept it as-is,
    so a decode loop over a fixed batch skips the per-call packing."""
    __slots__ = ("arr", "n")

    def __init__(self, ranges: Sequence[Range]):
        self.n = len(ranges)
        self.arr = (Range * max(self.n, 1))(*ranges)

    def __len__(self):
        return self.n


def range_array(ranges: Sequence[Range]) -> RangeArray:
    return RangeArray(ranges)


def _batch(ranges, num_rows: int, chunk_tokens: int, flags: int, scale: float):
    if isinstance(ranges, RangeArray):
        b = Batch(num_rows, ranges.n, ctypes.cast(ranges.arr, ctypes.POINTER(Range)), chunk_tokens, flags, scale)
        return b, ranges
    arr = (Range * max(len(ranges), 1))(*ranges)
    b = Batch(num_rows, len(ranges), ctypes.cast(arr, ctypes.POINTER(Range)), chunk_tokens, flags, scale)
    return b, arr


OWN_STREAM = ctypes.c_void_p(-1).value  # DATTN_OWN_STREAM


class Store:
    """Paged bf16/fp32/fp64 KV block store on one GPU (dattn_store)."""

    def __init__(self, head_dim: int, num_q_heads: int, num_kv_heads: int, dtype: int = BF16,
                 page_tokens: int = 16, num_pages: int = 1024, max_seqs: int = 64,
                 max_pages_per_seq: Optional[int] = None, device: int = 0, scale: float = 0.0):
        if max_pages_per_seq is None:
            max_pages_per_seq = num_pages
        cfg = StoreConfig(head_dim, num_q_heads, num_kv_heads, scale, dtype, page_tokens,
                          num_pages, max_seqs, max_pages_per_seq, device)
        h = ctypes.c_void_p()
        check(lib.dattn_store_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self.cfg = cfg
        self.head_dim, self.num_q_heads, self.num_kv_heads = head_dim, num_q_heads, num_kv_heads
        self.dtype, self.page_tokens, self.device = dtype, page_tokens, device
        inf = self.info()
        self.padded_dim = inf.padded_dim
        self.record_elems = inf.record_elems
        self.record_bytes = inf.record_bytes
        self.elem_bytes = inf.elem_bytes

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib.dattn_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> StoreInfo:
        i = StoreInfo()
        check(lib.dattn_store_get_info(self._h, ctypes.byref(i)))
        return i

    def set_timing(self, enable: bool):
        check(lib.dattn_store_set_timing(self._h, 1 if enable else 0))

    def stats(self, reset: bool = False) -> Stats:
        st = Stats()
        check(lib.dattn_store_get_stats(self._h, 1 if reset else 0, ctypes.byref(st)))
        return st

    def stream(self) -> int:
        s = ctypes.c_void_p()
        check(lib.dattn_store_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    def set_stream(self, stream_ptr: Optional[int]):
        """cudaStream_t handle for all later work. 0 / None is the CUDA default
        stream (torch's default-stream handle); OWN_STREAM restores the store's
        own non-blocking stream."""
        check(lib.dattn_store_set_stream(self._h, stream_ptr))

    def synchronize(self):
        check(lib.dattn_store_synchronize(self._h))

    # --- block ledger ---
    def seq_create(self, tokens: int) -> int:
        out = ctypes.c_int32()
        check(lib.dattn_seq_create(self._h, tokens, ctypes.byref(out)))
        return out.value

    def seq_resize(self, seq: int, tokens: int):
        check(lib.dattn_seq_resize(self._h, seq, tokens))

    def seq_release(self, seq: int) -> int:
        n = ctypes.c_int64()
        check(lib.dattn_seq_release(self._h, seq, ctypes.byref(n)))
        return n.value

    def seq_tokens(self, seq: int) -> int:
        n = ctypes.c_int64()
        check(lib.dattn_seq_tokens(self._h, seq, ctypes.byref(n)))
        return n.value

    def block_table(self, seq: int):
        n = ctypes.c_int64()
        check(lib.dattn_seq_block_table(self._h, seq, None, 0, ctypes.byref(n)))
        arr = (ctypes.c_int32 * max(n.value, 1))()
        check(lib.dattn_seq_block_table(self._h, seq, ctypes.cast(arr, ctypes.c_void_p), n.value,
                                        ctypes.byref(n)))
        return list(arr[: n.value])

    # --- data ---
    def kv_write(self, seq: int, kv_head: int, tok0: int, k, v, src_dtype: int = F64):
        import numpy as np
        k = np.ascontiguousarray(k)
        v = np.ascontiguousarray(v)
        n, d = k.shape
        check(lib.dattn_kv_write(self._h, seq, kv_head, tok0, n, k.ctypes.data, v.ctypes.data,
                                 src_dtype, d))

    def kv_read(self, seq: int, kv_head: int, tok0: int, n: int):
        """Rows as float64 numpy arrays [n, padded_dim] (store dtype widened)."""
        import numpy as np
        npdt = {BF16: np.uint16, F32: np.float32, F64: np.float64}[self.dtype]
        k = np.zeros((n, self.padded_dim), dtype=npdt)
        v = np.zeros((n, self.padded_dim), dtype=npdt)
        check(lib.dattn_kv_read(self._h, seq, kv_head, tok0, n, k.ctypes.data, v.ctypes.data))
        if self.dtype == BF16:
            k = (k.astype(np.uint32) << 16).view(np.float32)
            v = (v.astype(np.uint32) << 16).view(np.float32)
        return k.astype(np.float64), v.astype(np.float64)

    def kv_append(self, seqs: Sequence[int], k_new, v_new, mem: int = MEM_DEVICE):
        """Append one token to each sequence: k_new/v_new [n][num_kv_heads][padded_dim]."""
        arr = (ctypes.c_int32 * max(len(seqs), 1))(*seqs)
        check(lib.dattn_kv_append(self._h, len(seqs), ctypes.cast(arr, ctypes.c_void_p), ptr(k_new),
                                  ptr(v_new), mem))

    def synthetic_rows(self, logical_seqs: Sequence[int], logical_toks: Sequence[int], seed: int, k_dev, v_dev,
                       amp_k: float = 1.0, amp_v: float = 2.0):
        """K4's values of (logical_seqs[i], logical_toks[i]) as append rows
        [n][num_kv_heads][padded_dim] into device buffers."""
        n = len(logical_seqs)
        ls = (ctypes.c_uint32 * max(n, 1))(*logical_seqs)
        lt = (ctypes.c_int64 * max(n, 1))(*logical_toks)
        check(lib.dattn_kv_synthetic_rows(self._h, n, ctypes.cast(ls, ctypes.c_void_p), ctypes.cast(lt, ctypes.c_void_p),
                                          seed, amp_k, amp_v, ptr(k_dev), ptr(v_dev)))

    def fill_synthetic(self, seq: int, seed: int, logical_seq: int, logical_tok0: int = 0,
                       amp_k: float = 1.0, amp_v: float = 2.0):
        check(lib.dattn_kv_fill_synthetic(self._h, seq, seed, logical_seq, logical_tok0, amp_k, amp_v))

    def q_fill_synthetic(self, q_dev, rows: int, seed: int, row0: int = 0, amp_q: float = 1.0):
        check(lib.dattn_q_fill_synthetic(self._h, ptr(q_dev), rows, seed, row0, amp_q))

    # --- compute ---
    def decode(self, ranges: Sequence[Range], num_rows: int, q, out, row_partials=None,
               mem: int = MEM_DEVICE, chunk_tokens: int = 0, flags: int = 0, scale: float = 0.0):
        b, keep = _batch(ranges, num_rows, chunk_tokens, flags, scale)
        check(lib.dattn_decode(self._h, ctypes.byref(b), ptr(q), ptr(out), ptr(row_partials), mem))

    def micro_attention(self, ranges: Sequence[Range], num_rows: int, q_dev, partials_dev,
                        flags: int = 0, scale: float = 0.0):
        b, keep = _batch(ranges, num_rows, 0, flags, scale)
        check(lib.dattn_micro_attention(self._h, ctypes.byref(b), ptr(q_dev), ptr(partials_dev)))

    def merge(self, recs, rows: int, heads: int, n_uniform: int, row_mul: int, c_stride: int,
              out_recs=None, out_norm=None, row_begin=None):
        d = MergeDesc(rows, heads, ptr(row_begin), n_uniform, row_mul, c_stride)
        check(lib.dattn_merge_partials(self._h, ctypes.byref(d), ptr(recs), ptr(out_recs), ptr(out_norm)))

    # --- multi-GPU ---
    def comm_init(self, unique_id: bytes, rank: int, nranks: int):
        buf = ctypes.create_string_buffer(unique_id, 128)
        check(lib.dattn_comm_init(self._h, buf, rank, nranks))

    def comm_abort(self):
        """Make this rank's pending exchange polls give up (dattn_comm_abort)."""
        check(lib.dattn_comm_abort(self._h))

    def comm_info(self):
        """(rank, nranks, exchange) as NCCL reports the communicator; exchange
        1 = ncclAllGather + K3, 2 = K5 NVLink, 3 = MA-kernel push + K6."""
        r, n, x = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib.dattn_comm_info(self._h, ctypes.byref(r), ctypes.byref(n), ctypes.byref(x)))
        return r.value, n.value, x.value

    def decode_sharded(self, ranges: Sequence[Range], num_rows: int, q, out, mem: int = MEM_DEVICE,
                       chunk_tokens: int = 0, scale: float = 0.0):
        b, keep = _batch(ranges, num_rows, chunk_tokens, 0, scale)
        check(lib.dattn_decode_sharded(self._h, ctypes.byref(b), ptr(q), ptr(out), mem))

    def kv_send(self, seq: int, tok0: int, n: int, peer: int):
        """Migrate tokens [tok0, tok0+n) of every kv head of `seq` to `peer`."""
        check(lib.dattn_kv_send(self._h, seq, tok0, n, peer))

    def kv_recv(self, seq: int, tok0: int, n: int, peer: int):
        check(lib.dattn_kv_recv(self._h, seq, tok0, n, peer))

    def kv_pull(self, dst_seq: int, dst_tok0: int, src_rank: int, src_pages: Sequence[int]):
        """Copy whole pages of src_rank's pool into dst_seq at dst_tok0 over
        NVLink (copy engines, migration stream; returns at once)."""
        arr = (ctypes.c_int32 * max(len(src_pages), 1))(*src_pages)
        check(lib.dattn_kv_pull(self._h, dst_seq, dst_tok0, src_rank, ctypes.cast(arr, ctypes.c_void_p),
                                len(src_pages)))

    def migration_join(self, wait_host: bool = False):
        check(lib.dattn_kv_migration_join(self._h, 1 if wait_host else 0))


class Ledger:
    """The cluster block ledger + the decode loop's slot rule (include/dattn.h
    "block placement ledger"): one RManager ledger per instance
    (controlplane.cpp:38-79) and ensure_slot's overflow borrowing
    (simengine.cpp:318-354). Host-only; usable without a GPU."""

    def __init__(self, capacity_blocks: Sequence[int], block_tokens: int = 16):
        caps = (ctypes.c_int64 * len(capacity_blocks))(*capacity_blocks)
        h = ctypes.c_void_p()
        check(lib.dattn_ledger_create(len(capacity_blocks), caps, block_tokens, ctypes.byref(h)))
        self._h = h
        self.n_instances = len(capacity_blocks)
        self.block_tokens = block_tokens

    def close(self):
        if getattr(self, "_h", None):
            lib.dattn_ledger_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def admit(self, req: int, home: int, tokens: int) -> bool:
        a = ctypes.c_int()
        check(lib.dattn_ledger_admit(self._h, req, home, tokens, ctypes.byref(a)))
        return bool(a.value)

    def ensure_slot(self, req: int, allow_borrow: bool = True) -> int:
        """Instance holding the request's next token position, -1 if stalled."""
        i = ctypes.c_int()
        check(lib.dattn_ledger_ensure_slot(self._h, req, 1 if allow_borrow else 0, ctypes.byref(i)))
        return i.value

    def advance(self, req: int, tokens: int = 1):
        check(lib.dattn_ledger_advance(self._h, req, tokens))

    def step(self, reqs: Sequence[int], allow_borrow: bool = True):
        """ensure_slot for every request in order, then advance those with a
        slot by one token; returns the slot instances (-1: stalled)."""
        n = len(reqs)
        ra = (ctypes.c_int64 * max(n, 1))(*reqs)
        out = (ctypes.c_int * max(n, 1))()
        check(lib.dattn_ledger_step(self._h, n, ra, 1 if allow_borrow else 0, out))
        return list(out[:n])

    def release(self, req: int) -> int:
        f = ctypes.c_int64()
        check(lib.dattn_ledger_release(self._h, req, ctypes.byref(f)))
        return f.value

    def instance(self, i: int):
        """(capacity, used, free) blocks of instance i."""
        c, u, f = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(lib.dattn_ledger_instance(self._h, i, ctypes.byref(c), ctypes.byref(u), ctypes.byref(f)))
        return c.value, u.value, f.value

    def free_blocks(self, i: int) -> int:
        return self.instance(i)[2]

    def request(self, req: int):
        """(home, ctx tokens, held blocks)."""
        h, c, b = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
        check(lib.dattn_ledger_request(self._h, req, ctypes.byref(h), ctypes.byref(c), ctypes.byref(b)))
        return h.value, c.value, b.value

    def blocks(self, req: int, inst: int) -> int:
        n = ctypes.c_int64()
        check(lib.dattn_ledger_blocks(self._h, req, inst, ctypes.byref(n)))
        return n.value

    def segments(self, req: int):
        """[(instance, tok_begin, tok_end)] of positions [0, ctx), block order."""
        n = ctypes.c_int()
        check(lib.dattn_ledger_segments(self._h, req, 0, None, None, None, ctypes.byref(n)))
        k = n.value
        inst = (ctypes.c_int * max(k, 1))()
        lo = (ctypes.c_int64 * max(k, 1))()
        hi = (ctypes.c_int64 * max(k, 1))()
        check(lib.dattn_ledger_segments(self._h, req, k, inst, lo, hi, ctypes.byref(n)))
        return [(inst[i], lo[i], hi[i]) for i in range(k)]

    def borrowed(self) -> int:
        n = ctypes.c_int64()
        check(lib.dattn_ledger_borrowed(self._h, ctypes.byref(n)))
        return n.value


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib.dattn_comm_unique_id(buf))
    return buf.raw


def verify_attention(trials: int, seed: int, tolerance: float):
    """kvs_verify_attention (kvsched.h:56-62) on the GPU path. Returns (report, pass)."""
    rep = ctypes.c_void_p()
    ok = ctypes.c_int(-1)
    check(lib.dattn_verify_attention(trials, seed, tolerance, ctypes.byref(rep), ctypes.byref(ok)))
    text = ctypes.string_at(rep.value).decode()
    lib.dattn_string_free(rep)
    return text, bool(ok.value)


from .sharding import plan_rank_ranges, placement_from_moves, RankRange  # noqa: E402,F401
