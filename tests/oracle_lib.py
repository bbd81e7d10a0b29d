"""ctypes bindings for the TEST-INFRASTRUCTURE libraries under oracle/:

* oracle/build/libouro_oracle.so -- the CPU restatement (the checker);
* oracle/_ref/libouro_refconfig.so -- the reference's own proj/src/config.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use this.
"""
import ctypes as C
import os
import subprocess

from paper_2504_18211_b200._abi import (ChurnResult, Config, Digest, Geometry, ScriptStep, Stats,
                                        make_steps)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "build", "libouro_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libouro_refconfig.so")

_OR = None
_REF = None


class TrialOut(C.Structure):
    _fields_ = [("alloc_ms", C.c_double * 64), ("free_ms", C.c_double * 64),
                ("ok_allocs", C.c_uint64), ("failed_allocs", C.c_uint64),
                ("verified", C.c_uint32), ("threads", C.c_uint32)]


def build_oracle():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "build/libouro_oracle.so"], check=True)


def oracle():
    global _OR
    if _OR is None:
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = C.CDLL(ORACLE_SO)
        P, u8, u32, u64, i32 = C.c_void_p, C.c_uint8, C.c_uint32, C.c_uint64, C.c_int32
        sig = {
            "orc_config_validate": (i32, [C.POINTER(Config), C.c_char_p, C.c_size_t]),
            "orc_config_geometry": (i32, [C.POINTER(Config), C.POINTER(Geometry)]),
            "orc_variant_name": (C.c_char_p, [u8, u8]),
            "orc_variant_from_name": (C.c_int, [C.c_char_p, C.POINTER(u8), C.POINTER(u8)]),
            "orc_size_class": (i32, [C.POINTER(Config), u64, C.POINTER(u32)]),
            "orc_handle_encode": (i32, [C.POINTER(Config), u32, u32, C.POINTER(u32)]),
            "orc_handle_decode": (i32, [C.POINTER(Config), u32, C.POINTER(u32), C.POINTER(u32)]),
            "orc_backoff_ns": (u64, [u8, u32, u32, u32]),
            "orc_pattern_word": (u64, [u64, u64, u32, u64]),
            "orc_mix64": (u64, [u64]),
            "orc_heap_create": (i32, [C.POINTER(Config), C.POINTER(P)]),
            "orc_heap_destroy": (None, [P]),
            "orc_alloc_group": (i32, [P, u32, C.POINTER(u64), C.POINTER(u64), C.POINTER(i32)]),
            "orc_free_group": (i32, [P, u32, C.POINTER(u64), C.POINTER(i32)]),
            "orc_alloc_coalesced": (i32, [P, u32, u64, C.POINTER(u64), C.POINTER(i32)]),
            "orc_run_script": (i32, [P, C.POINTER(ScriptStep), u32, C.POINTER(u64), C.POINTER(i32)]),
            "orc_page_region": (i32, [P, u32, C.POINTER(u64), C.POINTER(u64)]),
            "orc_stats": (i32, [P, C.POINTER(Stats)]),
            "orc_digest": (i32, [P, C.POINTER(Digest)]),
            "orc_queue_ops": (u64, [P]),
            "orc_pool_dequeues": (u64, [P]),
            "orc_chunk_assign": (i32, [P, u32, u32, C.POINTER(u32)]),
            "orc_chunk_acquire": (i32, [P, u32, C.POINTER(u32)]),
            "orc_chunk_release": (i32, [P, u32, u32, C.POINTER(u32)]),
            "orc_chunk_unassign": (i32, [P, u32]),
            "orc_chunk_state": (i32, [P, u32, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32), C.POINTER(u64)]),
            "orc_qt_new": (i32, [u8, u64, u32, u64, C.POINTER(P)]),
            "orc_qt_destroy": (None, [P]),
            "orc_qt_enqueue": (i32, [P, u32]),
            "orc_qt_dequeue": (i32, [P, C.POINTER(u32)]),
            "orc_qt_len": (u64, [P]),
            "orc_qt_pool_len": (u64, [P]),
            "orc_qt_seg_live": (u64, [P]),
            "orc_qt_mt_churn": (i32, [P, u32, u32, u32, C.POINTER(u32), C.c_double]),
            "orc_active_mask": (i32, [u32, C.POINTER(i32), u32, C.POINTER(u64)]),
            "orc_bench_trial": (i32, [P, u64, u64, C.POINTER(u32), u32, u32, u64, C.POINTER(TrialOut)]),
            "orc_churn": (i32, [P, u64, u32, u32, u64, u32, C.POINTER(u64), C.POINTER(ChurnResult),
                                C.POINTER(C.c_double)]),
            "orc_free_all": (i32, [P, u64, C.POINTER(u64)]),
            "orc_alloc_slots": (i32, [P, u64, u64, C.POINTER(u32), u32, C.POINTER(u64), C.POINTER(u64)]),
            "orc_free_slots": (i32, [P, u64, C.POINTER(u64), u32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _OR = L
    return _OR


def ref():
    """The reference's own config.cpp (None if it was never built here)."""
    global _REF
    if _REF is None:
        if not os.path.exists(REF_SO):
            if os.path.exists("/root/reference/proj/src/config.cpp"):
                subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
            if not os.path.exists(REF_SO):
                return None
        L = C.CDLL(REF_SO)
        L.ref_validate.restype = C.c_int
        L.ref_validate.argtypes = [C.POINTER(Config), C.c_char_p, C.c_size_t]
        L.ref_default.argtypes = [C.POINTER(Config)]
        L.ref_num_chunks.restype = C.c_uint32
        L.ref_num_chunks.argtypes = [C.POINTER(Config)]
        L.ref_max_pages_per_chunk.restype = C.c_uint32
        L.ref_max_pages_per_chunk.argtypes = [C.POINTER(Config)]
        L.ref_variant_name.restype = C.c_int
        L.ref_variant_name.argtypes = [C.c_uint8, C.c_uint8, C.c_char_p, C.c_size_t]
        L.ref_variant_from_name.restype = C.c_int
        L.ref_variant_from_name.argtypes = [C.c_char_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint8)]
        L.ref_all_variants.restype = C.c_int
        L.ref_all_variants.argtypes = [C.POINTER(C.c_uint8), C.POINTER(C.c_uint8)]
        L.ref_layout.argtypes = [C.POINTER(C.c_uint64)]
        _REF = L
    return _REF


class OHeap:
    """Oracle heap (thread-safe for group-of-1 ops)."""

    def __init__(self, cfg: Config):
        self.L = oracle()
        h = C.c_void_p()
        st = self.L.orc_heap_create(C.byref(cfg), C.byref(h))
        if st != 0:
            raise ValueError(f"orc_heap_create: {st}")
        self.h = h
        self.cfg = cfg

    def close(self):
        if self.h:
            self.L.orc_heap_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def alloc(self, sizes):
        n = len(sizes)
        s = (C.c_uint64 * n)(*sizes)
        off = (C.c_uint64 * n)()
        st = (C.c_int32 * n)()
        assert self.L.orc_alloc_group(self.h, n, s, off, st) == 0
        return list(off), list(st)

    def free(self, offs):
        n = len(offs)
        o = (C.c_uint64 * n)(*offs)
        st = (C.c_int32 * n)()
        assert self.L.orc_free_group(self.h, n, o, st) == 0
        return list(st)

    def alloc_coalesced(self, n, nbytes):
        off = (C.c_uint64 * n)()
        st = (C.c_int32 * n)()
        assert self.L.orc_alloc_coalesced(self.h, n, nbytes, off, st) == 0
        return list(off), list(st)

    def alloc_slots(self, n, nbytes=0, sizes=None, group=32):
        """n slots in warp groups (slot order): (offsets array, success count)."""
        out = (C.c_uint64 * n)()
        ok = C.c_uint64()
        sz = None
        if sizes is not None:
            sz = (C.c_uint32 * n)(*sizes)
        assert self.L.orc_alloc_slots(self.h, n, nbytes, sz, group, out, C.byref(ok)) == 0
        return out, ok.value

    def free_slots(self, offs, group=32):
        assert self.L.orc_free_slots(self.h, len(offs), offs, group) == 0

    def churn(self, n, round_begin, rounds, seed, threads=1, slots=None):
        """orc_churn over n slots; returns (slots array, ChurnResult)."""
        if slots is None:
            slots = (C.c_uint64 * n)(*([2 ** 64 - 1] * n))
        res, ms = ChurnResult(), C.c_double()
        assert self.L.orc_churn(self.h, n, round_begin, rounds, seed, threads, slots, C.byref(res), C.byref(ms)) == 0
        return slots, res

    def free_all(self, slots):
        assert self.L.orc_free_all(self.h, len(slots), slots) == 0

    def run_script(self, steps):
        arr = make_steps(steps)
        n = len(steps)
        off = (C.c_uint64 * (n * 32))()
        st = (C.c_int32 * (n * 32))()
        assert self.L.orc_run_script(self.h, arr, n, off, st) == 0
        return list(off), list(st)

    def stats(self) -> Stats:
        s = Stats()
        self.L.orc_stats(self.h, C.byref(s))
        return s

    def digest(self) -> Digest:
        d = Digest()
        self.L.orc_digest(self.h, C.byref(d))
        return d

    def page_region(self, handle):
        off, ln = C.c_uint64(), C.c_uint64()
        st = self.L.orc_page_region(self.h, handle, C.byref(off), C.byref(ln))
        return st, off.value, ln.value

    def queue_ops(self):
        return self.L.orc_queue_ops(self.h)

    def pool_dequeues(self):
        return self.L.orc_pool_dequeues(self.h)
