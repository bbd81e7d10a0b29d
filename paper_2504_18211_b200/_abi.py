"""ctypes mirrors of the POD types in include/ouro.h (shared by the product
bindings and the test-side oracle bindings)."""
import ctypes as C

MAX_CLASSES = 32

# ouro_status (include/ouro.h); 1..6 = /root/reference/proj/include/ouro/errors.hpp:11-46
OK = 0
ERR_CONFIG = 1
ERR_INVALID_HANDLE = 2
ERR_DOUBLE_FREE = 3
ERR_RANGE = 4
ERR_TIMEOUT = 5
ERR_CORRUPTION = 6
ERR_OOM = 7
ERR_TOO_LARGE = 8
ERR_CUDA = 9
ERR_FULL = 10
ERR_EMPTY = 11
ERR_CHUNK_FULL = 12
ERR_ALREADY_ASSIGNED = 13
ERR_VERIFICATION = 14
ERR_USAGE = 15

STATUS_NAMES = {
    0: "Ok", 1: "ConfigError", 2: "InvalidHandle", 3: "DoubleFree", 4: "RangeError",
    5: "Timeout", 6: "Corruption", 7: "OutOfMemory", 8: "TooLarge", 9: "CudaError",
    10: "Full", 11: "Empty", 12: "ChunkFull", 13: "AlreadyAssigned",
    14: "VerificationFailed", 15: "UsageError",
}


class Config(C.Structure):
    """ouro_config == ouro::HeapConfig (config.hpp:26-38), 48 bytes."""
    _fields_ = [
        ("heap_bytes", C.c_uint64), ("chunk_bytes", C.c_uint64),
        ("min_page_bytes", C.c_uint64), ("max_page_bytes", C.c_uint64),
        ("queue_flavor", C.c_uint8), ("allocator_kind", C.c_uint8),
        ("backoff", C.c_uint8), ("reserved0", C.c_uint8),
        ("max_retries", C.c_uint32), ("sleep_base_ns", C.c_uint32), ("sleep_cap_ns", C.c_uint32),
    ]


class Geometry(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "num_chunks", "max_pages_per_chunk", "num_classes", "page_bits", "chunk_bits",
        "gen_bits", "bitmap_words", "reserved0")]


class ClassStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "page_bytes", "pages_per_chunk", "chunks", "live_pages", "queue_len", "queued_live",
        "seg_live", "seg_hwm", "retries", "ooms")]


class Stats(C.Structure):
    _fields_ = [
        ("num_classes", C.c_uint32), ("num_chunks", C.c_uint32),
        ("sticky_first", C.c_uint32), ("sticky_mask", C.c_uint32),
        ("pool_len", C.c_uint64), ("stale_drops", C.c_uint64), ("double_frees", C.c_uint64),
        ("invalid_frees", C.c_uint64), ("bad_sizes", C.c_uint64), ("timeouts", C.c_uint64),
        ("corruptions", C.c_uint64), ("cls", ClassStats * MAX_CLASSES),
    ]


class Digest(C.Structure):
    _fields_ = [
        ("num_chunks", C.c_uint32), ("num_classes", C.c_uint32),
        ("partition_ok", C.c_uint32), ("sticky_mask", C.c_uint32),
        ("live_pages", C.c_uint64), ("unassigned_chunks", C.c_uint64),
        ("header_hash", C.c_uint64), ("queue_hash", C.c_uint64),
        ("class_chunks", C.c_uint64 * MAX_CLASSES),
        ("class_queued_live", C.c_uint64 * MAX_CLASSES),
        ("class_live_pages", C.c_uint64 * MAX_CLASSES),
    ]

    def as_dict(self):
        k = self.num_classes
        return {
            "num_chunks": self.num_chunks, "num_classes": k,
            "partition_ok": self.partition_ok, "sticky_mask": self.sticky_mask,
            "live_pages": self.live_pages, "unassigned_chunks": self.unassigned_chunks,
            "header_hash": self.header_hash, "queue_hash": self.queue_hash,
            "class_chunks": list(self.class_chunks[:k]),
            "class_queued_live": list(self.class_queued_live[:k]),
            "class_live_pages": list(self.class_live_pages[:k]),
        }


class ScriptStep(C.Structure):
    _fields_ = [("op", C.c_uint32), ("lane_mask", C.c_uint32), ("arg", C.c_uint64 * 32)]


class TrialConfig(C.Structure):
    _fields_ = [
        ("num_allocations", C.c_uint64), ("allocation_bytes", C.c_uint64),
        ("sizes", C.POINTER(C.c_uint32)), ("iterations", C.c_uint32), ("reserved0", C.c_uint32),
        ("seed", C.c_uint64),
    ]


class TrialResult(C.Structure):
    _fields_ = [
        ("alloc_ms", C.c_double * 64), ("free_ms", C.c_double * 64),
        ("write_ms", C.c_double * 64), ("verify_ms", C.c_double * 64),
        ("iterations", C.c_uint32), ("verified", C.c_uint32),
        ("ok_allocs", C.c_uint64), ("failed_allocs", C.c_uint64),
        ("mean_all_ms", C.c_double), ("mean_subsequent_ms", C.c_double),
        ("mean_subsequent_free_ms", C.c_double),
        ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
    ]


class AuditResult(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "live", "out_of_heap", "misaligned", "overlaps", "not_marked", "bytes")]


class ChurnResult(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "mallocs_ok", "mallocs_failed", "frees", "reused", "check_failures")]


MAX_DEVICES = 16


class MultiResult(C.Structure):
    _fields_ = [("ndev", C.c_uint32), ("verified", C.c_uint32), ("pairs_total", C.c_uint64),
                ("max_ms", C.c_double), ("pairs_per_s", C.c_double),
                ("dev_ms", C.c_double * MAX_DEVICES), ("dev_pairs", C.c_uint64 * MAX_DEVICES)]


_VARIANT_NAMES = {(0, 0): "page", (1, 0): "chunk", (0, 1): "va-page", (1, 1): "va-chunk",
                  (0, 2): "vl-page", (1, 2): "vl-chunk"}


def variant_name_of(kind: int, flavor: int) -> str:
    """variant_name (config.cpp:44-52) without loading the library (the reference
    bench arm runs on a host without the CUDA build)."""
    return _VARIANT_NAMES[(int(kind), int(flavor))]


def make_steps(steps):
    """steps: list of (op, lane_mask, args[32]) -> ctypes array of ScriptStep."""
    arr = (ScriptStep * max(1, len(steps)))()
    for i, (op, mask, args) in enumerate(steps):
        arr[i].op = op
        arr[i].lane_mask = mask
        for j in range(32):
            arr[i].arg[j] = int(args[j]) if j < len(args) else 0
    return arr
