"""paper_2504_18211_b200 -- B200-native Ouroboros-style device allocator.

Python mirror of the reference's C++ API (namespace ``ouro``,
/root/reference/proj/include/ouro/{config,errors}.hpp) over the C-ABI in
include/ouro.h, implemented by the in-tree ``libouro_b200.so`` (sm_100a).

  reference                              here
  -------------------------------------  ---------------------------------------
  ouro::HeapConfig (config.hpp:26-52)    HeapConfig (same fields and defaults)
  HeapConfig::validate (config.cpp:16)   HeapConfig.validate() -> ConfigError
  QueueFlavor/AllocatorKind/Backoff...   QueueFlavor / AllocatorKind / BackoffPolicy
  Variant, kAllVariants (config.hpp:55)  Variant, ALL_VARIANTS
  variant_name / variant_from_name       variant_name / variant_from_name
  error classes (errors.hpp:11-46)       ConfigError ... CorruptionError
  new_arena / alloc / dealloc (SPEC)     Heap (device heap; in-kernel malloc/free)

There is no CPU fallback: a missing or unloadable library raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

from . import _abi
from ._abi import (AuditResult, ChurnResult, Config, Digest, Geometry, MultiResult, ScriptStep, Stats,
                   TrialConfig, TrialResult, make_steps)

__all__ = [
    "HeapConfig", "QueueFlavor", "AllocatorKind", "BackoffPolicy", "Variant", "ALL_VARIANTS",
    "variant_name", "variant_from_name", "Heap", "OuroError", "ConfigError",
    "InvalidHandleError", "DoubleFreeError", "RangeError", "TimeoutError_", "CorruptionError",
    "lib", "lib_path", "size_class", "backoff_ns", "multi_sweep",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib_path() -> str:
    # OURO_B200_LIB: an alternative in-tree build (compile-time experiments)
    return os.environ.get("OURO_B200_LIB") or os.path.join(_HERE, "libouro_b200.so")


def lib() -> C.CDLL:
    """Load libouro_b200.so (built by `make -C paper_2504_18211_b200`)."""
    global _LIB
    if _LIB is None:
        p = lib_path()
        if not os.path.exists(p):
            raise RuntimeError(f"libouro_b200.so not built ({p}); run __graft_entry__.build()")
        L = C.CDLL(p)
        _declare(L)
        _LIB = L
    return _LIB


def _declare(L):
    P, u8, u32, u64, i32 = C.c_void_p, C.c_uint8, C.c_uint32, C.c_uint64, C.c_int32
    sig = {
        "ouro_config_default": (i32, [C.POINTER(Config)]),
        "ouro_config_validate": (i32, [C.POINTER(Config), C.c_char_p, C.c_size_t]),
        "ouro_config_geometry": (i32, [C.POINTER(Config), C.POINTER(Geometry)]),
        "ouro_variant_name": (C.c_char_p, [u8, u8]),
        "ouro_variant_from_name": (C.c_int, [C.c_char_p, C.POINTER(u8), C.POINTER(u8)]),
        "ouro_size_class": (i32, [C.POINTER(Config), u64, C.POINTER(u32)]),
        "ouro_handle_encode": (i32, [C.POINTER(Config), u32, u32, C.POINTER(u32)]),
        "ouro_handle_decode": (i32, [C.POINTER(Config), u32, C.POINTER(u32), C.POINTER(u32)]),
        "ouro_backoff_ns": (u64, [u8, u32, u32, u32]),
        "ouro_heap_create": (i32, [C.POINTER(Config), C.c_int, C.POINTER(P)]),
        "ouro_heap_destroy": (i32, [P]),
        "ouro_heap_reset": (i32, [P, P]),
        "ouro_heap_get_view": (i32, [P, P, C.c_size_t]),
        "ouro_heap_view_size": (C.c_size_t, []),
        "ouro_heap_set_checks": (i32, [P, C.c_int]),
        "ouro_heap_set_spin_limit": (i32, [P, u64]),
        "ouro_heap_debug_add_count": (i32, [P, u32, C.c_int64]),
        "ouro_set_launch_shape": (i32, [C.c_int, C.c_int]),
        "ouro_heap_set_launch_shape": (i32, [P, C.c_int, C.c_int]),
        "ouro_multi_sweep": (i32, [C.POINTER(Config), u32, C.POINTER(C.c_int), u64, C.POINTER(u32), u32, u32, u32,
                                   C.POINTER(MultiResult)]),
        "ouro_debug_counters": (i32, [C.POINTER(u64), C.c_int]),
        "ouro_heap_config": (i32, [P, C.POINTER(Config), C.POINTER(Geometry)]),
        "ouro_heap_base": (u64, [P]),
        "ouro_page_region": (i32, [P, u32, C.POINTER(u64), C.POINTER(u64)]),
        "ouro_heap_stats": (i32, [P, C.POINTER(Stats), P]),
        "ouro_heap_digest": (i32, [P, C.POINTER(Digest), P]),
        "ouro_heap_last_error": (i32, [P, C.POINTER(u32), C.POINTER(u32), C.c_int]),
        "ouro_launch_alloc": (i32, [P, u64, u64, P, P, P]),
        "ouro_launch_alloc_u16": (i32, [P, u64, P, P, P]),
        "ouro_heap_queue_links": (i32, [P, u32, C.POINTER(u64)]),
        "ouro_heap_vl_ring": (i32, [P, u32, C.POINTER(u64)]),
        "ouro_launch_free": (i32, [P, u64, P, P]),
        "ouro_launch_write": (i32, [P, u64, P, u64, u32, P]),
        "ouro_launch_verify": (i32, [P, u64, P, u64, u32, P, P]),
        "ouro_launch_count": (i32, [P, u64, P, P, P]),
        "ouro_audit": (i32, [P, u64, P, C.POINTER(AuditResult), P]),
        "ouro_launch_churn": (i32, [P, u64, u32, u32, u64, P, P, P]),
        "ouro_run_script": (i32, [P, C.POINTER(ScriptStep), u32, C.POINTER(u64), C.POINTER(i32)]),
        "ouro_run_trial": (i32, [P, C.POINTER(TrialConfig), C.POINTER(TrialResult)]),
        "ouro_trial_means": (i32, [C.POINTER(C.c_double), u32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "ouro_atomic_peak": (i32, [C.c_int, C.c_int, C.POINTER(C.c_double)]),
        "ouro_status_name": (C.c_char_p, [i32]),
        "ouro_build_info": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name, None)
        if f is None:  # an older experiment build (OURO_B200_LIB); tests/test_abi.py checks the product
            continue
        f.restype = res
        f.argtypes = args


# ---------------------------------------------------------------- errors ----
class OuroError(RuntimeError):
    status = -1


class ConfigError(OuroError):          # errors.hpp:11
    status = _abi.ERR_CONFIG


class InvalidHandleError(OuroError):   # errors.hpp:17
    status = _abi.ERR_INVALID_HANDLE


class DoubleFreeError(OuroError):      # errors.hpp:24
    status = _abi.ERR_DOUBLE_FREE


class RangeError(OuroError):           # errors.hpp:30
    status = _abi.ERR_RANGE


class TimeoutError_(OuroError):        # errors.hpp:36
    status = _abi.ERR_TIMEOUT


class CorruptionError(OuroError):      # errors.hpp:43
    status = _abi.ERR_CORRUPTION


class CudaError(OuroError):
    status = _abi.ERR_CUDA


_BY_STATUS = {c.status: c for c in (ConfigError, InvalidHandleError, DoubleFreeError, RangeError,
                                    TimeoutError_, CorruptionError, CudaError)}


def check(status: int, what: str = "") -> None:
    if status != _abi.OK:
        cls = _BY_STATUS.get(status, OuroError)
        raise cls(f"{what}: {_abi.STATUS_NAMES.get(status, status)}")


# ------------------------------------------------------------ config ----
class QueueFlavor(enum.IntEnum):      # config.hpp:17
    Array = 0
    VirtualArray = 1
    VirtualList = 2


class AllocatorKind(enum.IntEnum):    # config.hpp:21
    Page = 0
    Chunk = 1


class BackoffPolicy(enum.IntEnum):    # config.hpp:24
    FenceRetry = 0
    SleepRetry = 1


@dataclass
class HeapConfig:
    """ouro::HeapConfig (config.hpp:26-52): same fields, same defaults."""
    heap_bytes: int = 64 << 20
    chunk_bytes: int = 64 << 10
    min_page_bytes: int = 16
    max_page_bytes: int = 8192
    queue_flavor: QueueFlavor = QueueFlavor.Array
    allocator_kind: AllocatorKind = AllocatorKind.Page
    backoff: BackoffPolicy = BackoffPolicy.FenceRetry
    max_retries: int = 64
    sleep_base_ns: int = 100
    sleep_cap_ns: int = 100_000

    def to_c(self) -> Config:
        return Config(self.heap_bytes, self.chunk_bytes, self.min_page_bytes, self.max_page_bytes,
                      int(self.queue_flavor), int(self.allocator_kind), int(self.backoff), 0,
                      self.max_retries, self.sleep_base_ns, self.sleep_cap_ns)

    def validate(self) -> None:
        """Throws ConfigError exactly where HeapConfig::validate does (config.cpp:16-42)."""
        msg = C.create_string_buffer(256)
        c = self.to_c()
        st = lib().ouro_config_validate(C.byref(c), msg, 256)
        if st != _abi.OK:
            raise ConfigError(msg.value.decode())

    def num_chunks(self) -> int:          # config.hpp:45-47
        return (self.heap_bytes // self.chunk_bytes) & 0xFFFFFFFF

    def max_pages_per_chunk(self) -> int:  # config.hpp:49-51
        return (self.chunk_bytes // self.min_page_bytes) & 0xFFFFFFFF

    def geometry(self) -> Geometry:
        g = Geometry()
        c = self.to_c()
        check(lib().ouro_config_geometry(C.byref(c), C.byref(g)), "geometry")
        return g

    @property
    def variant(self) -> "Variant":
        return Variant(AllocatorKind(self.allocator_kind), QueueFlavor(self.queue_flavor))


@dataclass(frozen=True)
class Variant:                        # config.hpp:55-60
    kind: AllocatorKind
    flavor: QueueFlavor


ALL_VARIANTS = (                      # kAllVariants, config.hpp:62-69
    Variant(AllocatorKind.Page, QueueFlavor.Array),
    Variant(AllocatorKind.Chunk, QueueFlavor.Array),
    Variant(AllocatorKind.Page, QueueFlavor.VirtualArray),
    Variant(AllocatorKind.Chunk, QueueFlavor.VirtualArray),
    Variant(AllocatorKind.Page, QueueFlavor.VirtualList),
    Variant(AllocatorKind.Chunk, QueueFlavor.VirtualList),
)


def variant_name(v: Variant) -> str:          # config.cpp:44-52
    return lib().ouro_variant_name(int(v.kind), int(v.flavor)).decode()


def variant_from_name(name: str):             # config.cpp:54-59
    k, f = C.c_uint8(), C.c_uint8()
    if lib().ouro_variant_from_name(name.encode(), C.byref(k), C.byref(f)):
        return Variant(AllocatorKind(k.value), QueueFlavor(f.value))
    return None


def size_class(cfg: HeapConfig, nbytes: int) -> int:
    """size_class_of: class index; raises OuroError(TooLarge)."""
    k = C.c_uint32()
    c = cfg.to_c()
    st = lib().ouro_size_class(C.byref(c), nbytes, C.byref(k))
    if st != _abi.OK:
        e = OuroError(f"size_class({nbytes}): {_abi.STATUS_NAMES.get(st)}")
        e.status = st
        raise e
    return k.value


def backoff_ns(policy: int, attempt: int, base_ns: int = 100, cap_ns: int = 100_000) -> int:
    return lib().ouro_backoff_ns(policy, attempt, base_ns, cap_ns)


# -------------------------------------------------------------- heap ----
def _ptr(x):
    """Device pointer of a torch tensor, int, or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


class Heap:
    """A device heap (new_arena + allocator).

    Kernels call ouro_malloc / ouro_free on it (include/ouro_device.cuh); the
    methods here are the host side: batch launchers for the paper's driver
    phases, stats, the canonical digest, audits and op scripts."""

    def __init__(self, cfg: HeapConfig, device: int = 0):
        self.cfg = cfg
        self.device = device
        cfg.validate()
        h = C.c_void_p()
        c = cfg.to_c()
        check(lib().ouro_heap_create(C.byref(c), device, C.byref(h)), "ouro_heap_create")
        self._h = h
        self.base = lib().ouro_heap_base(h)
        self.geometry = cfg.geometry()

    def close(self):
        if getattr(self, "_h", None):
            lib().ouro_heap_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def set_checks(self, on: bool = True):
        """Debug mode: verify queue/bitmap invariants on every device op."""
        check(lib().ouro_heap_set_checks(self._h, int(on)), "set_checks")

    def set_spin_limit(self, limit: int):
        """Bounded device waits: spins before TimeoutError (errors.hpp:35-39)."""
        check(lib().ouro_heap_set_spin_limit(self._h, limit), "set_spin_limit")

    def debug_add_count(self, qi: int, delta: int):
        """Test-only fault injection into queue qi's occupancy count."""
        check(lib().ouro_heap_debug_add_count(self._h, qi, delta), "debug_add_count")

    def queue_links(self, qi: int):
        """Debug: (count, head ticket, vl_head, vl_tail) of queue qi."""
        out = (C.c_uint64 * 4)()
        check(lib().ouro_heap_queue_links(self._h, qi, out), "queue_links")
        return tuple(out)

    def vl_ring(self, qi: int):
        """Debug: the dequeue-side VirtualList ring of queue qi (256 links)."""
        out = (C.c_uint64 * 256)()
        check(lib().ouro_heap_vl_ring(self._h, qi, out), "vl_ring")
        return list(out)

    def reset(self, stream=None):
        check(lib().ouro_heap_reset(self._h, _stream(stream)), "reset")

    def view_bytes(self) -> bytes:
        n = lib().ouro_heap_view_size()
        buf = C.create_string_buffer(n)
        check(lib().ouro_heap_get_view(self._h, buf, n), "view")
        return buf.raw

    def stats(self, stream=None) -> Stats:
        s = Stats()
        check(lib().ouro_heap_stats(self._h, C.byref(s), _stream(stream)), "stats")
        return s

    def digest(self, stream=None) -> Digest:
        d = Digest()
        check(lib().ouro_heap_digest(self._h, C.byref(d), _stream(stream)), "digest")
        return d

    def last_error(self, clear=False):
        a, b = C.c_uint32(), C.c_uint32()
        check(lib().ouro_heap_last_error(self._h, C.byref(a), C.byref(b), int(clear)), "last_error")
        return a.value, b.value

    def page_region(self, handle: int):
        off, ln = C.c_uint64(), C.c_uint64()
        st = lib().ouro_page_region(self._h, handle, C.byref(off), C.byref(ln))
        check(st, "page_region")
        return off.value, ln.value

    def set_launch_shape(self, block_threads=256, waves=0):
        """Launch shape of this heap's alloc/free/churn launchers (ouro_heap_set_launch_shape)."""
        check(lib().ouro_heap_set_launch_shape(self._h, block_threads, waves), "set_launch_shape")

    # ---- driver phases (device buffers: torch tensors or raw pointers) ----
    def _check_buf(self, x, n, what, dtypes=None, min_elems=None):
        """Tensors handed to the launchers: on this heap's device, of an accepted
        dtype, with room for n elements (the kernels index [0, n) unchecked)."""
        if x is None or isinstance(x, int):
            return
        dev = getattr(x, "device", None)
        if dev is not None and (dev.type != "cuda" or (dev.index if dev.index is not None else 0) != self.device):
            raise ValueError(f"{what}: tensor on {dev}, heap on cuda:{self.device}")
        if dtypes is not None and str(x.dtype).replace("torch.", "") not in dtypes:
            raise ValueError(f"{what}: dtype {x.dtype} not one of {sorted(dtypes)}")
        if x.numel() < (n if min_elems is None else min_elems):
            raise ValueError(f"{what}: {x.numel()} elements < {n}")

    def launch_alloc(self, n, out_ptrs, size=0, sizes=None, stream=None):
        """sizes: optional device array of per-slot request sizes, int32 or int16/uint16."""
        self._check_buf(out_ptrs, n, "out_ptrs", {"int64", "uint64"})
        self._check_buf(sizes, n, "sizes", {"int32", "uint32", "int16", "uint16"})
        if sizes is not None and getattr(sizes, "element_size", lambda: 4)() == 2:
            check(lib().ouro_launch_alloc_u16(self._h, n, _ptr(sizes), _ptr(out_ptrs), _stream(stream)), "alloc")
            return
        check(lib().ouro_launch_alloc(self._h, n, size, _ptr(sizes), _ptr(out_ptrs), _stream(stream)), "alloc")

    def launch_free(self, n, ptrs, stream=None):
        self._check_buf(ptrs, n, "ptrs", {"int64", "uint64"})
        check(lib().ouro_launch_free(self._h, n, _ptr(ptrs), _stream(stream)), "free")

    def launch_write(self, n, ptrs, seed, iteration, stream=None):
        self._check_buf(ptrs, n, "ptrs", {"int64", "uint64"})
        check(lib().ouro_launch_write(self._h, n, _ptr(ptrs), seed, iteration, _stream(stream)), "write")

    def launch_verify(self, n, ptrs, seed, iteration, result, stream=None):
        self._check_buf(ptrs, n, "ptrs", {"int64", "uint64"})
        self._check_buf(result, 2, "result", {"int64", "uint64"})
        check(lib().ouro_launch_verify(self._h, n, _ptr(ptrs), seed, iteration, _ptr(result),
                                       _stream(stream)), "verify")

    def launch_count(self, n, ptrs, count, stream=None):
        self._check_buf(ptrs, n, "ptrs", {"int64", "uint64"})
        self._check_buf(count, 1, "count", {"int64", "uint64"})
        check(lib().ouro_launch_count(self._h, n, _ptr(ptrs), _ptr(count), _stream(stream)), "count")

    def launch_churn(self, n, round_begin, rounds, seed, slots, result, stream=None):
        self._check_buf(slots, n, "slots", {"int64", "uint64"})
        self._check_buf(result, 5, "result", {"int64", "uint64"})
        check(lib().ouro_launch_churn(self._h, n, round_begin, rounds, seed, _ptr(slots), _ptr(result),
                                      _stream(stream)), "churn")

    def audit(self, n, ptrs, stream=None) -> AuditResult:
        self._check_buf(ptrs, n, "ptrs", {"int64", "uint64"})
        r = AuditResult()
        check(lib().ouro_audit(self._h, n, _ptr(ptrs), C.byref(r), _stream(stream)), "audit")
        return r

    def run_script(self, steps):
        arr = make_steps(steps)
        n = len(steps)
        off = (C.c_uint64 * (n * 32))()
        st = (C.c_int32 * (n * 32))()
        check(lib().ouro_run_script(self._h, arr, n, off, st), "run_script")
        return list(off), list(st)

    def run_trial(self, n, nbytes=0, sizes=None, iterations=10, seed=1) -> TrialResult:
        tc = TrialConfig()
        tc.num_allocations = n
        tc.allocation_bytes = nbytes
        keep = None
        if sizes is not None:
            keep = (C.c_uint32 * n)(*sizes)
            tc.sizes = C.cast(keep, C.POINTER(C.c_uint32))
        tc.iterations = iterations
        tc.seed = seed
        r = TrialResult()
        check(lib().ouro_run_trial(self._h, C.byref(tc), C.byref(r)), "run_trial")
        return r


def multi_sweep(cfg: HeapConfig, devices, threads_per_device, sizes, warmup=1, steps=3) -> MultiResult:
    """ouro_multi_sweep: one host thread and one heap per entry of `devices` (devices may
    repeat), every step runs the size sweep on all of them behind a host barrier;
    aggregate pairs/s = pairs over devices / the slowest device's alloc + free time."""
    devs = (C.c_int * len(devices))(*devices)
    sz = (C.c_uint32 * len(sizes))(*sizes)
    r = MultiResult()
    c = cfg.to_c()
    check(lib().ouro_multi_sweep(C.byref(c), len(devices), devs, threads_per_device, sz, len(sizes), warmup, steps,
                                 C.byref(r)), "multi_sweep")
    return r


def atomic_peak(device: int, mode: int) -> float:
    v = C.c_double()
    check(lib().ouro_atomic_peak(device, mode, C.byref(v)), "atomic_peak")
    return v.value
