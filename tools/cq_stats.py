"""Per-warp cq_alloc timeline of an OURO_STORM_STATS=1, OURO_CQ_BLOCK=0 build:
OURO_B200_LIB=exp_stats/cqstats.so python tools/cq_stats.py [size] [flavor] [heap_log2] [threads_log2]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

size = int(sys.argv[1]) if len(sys.argv) > 1 else 16
fl = int(sys.argv[2]) if len(sys.argv) > 2 else 0
heap = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 30)
n = 1 << (int(sys.argv[4]) if len(sys.argv) > 4 else 20)
L = ob.lib()
L.ouro_debug_counters.argtypes = [C.POINTER(C.c_uint64), C.c_int]
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
out = (C.c_uint64 * 32)()
with ob.Heap(ob.HeapConfig(heap, allocator_kind=ob.AllocatorKind(1), queue_flavor=ob.QueueFlavor(fl))) as h:
    for it in range(3):
        L.ouro_debug_counters(out, 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.launch_alloc(n, ptrs, size=size); b.record(); b.synchronize()
        L.ouro_debug_counters(out, 1)
        w = max(out[25], 1)
        print(f"size {size} fl {fl} alloc_us={a.elapsed_time(b) * 1000:.1f} calls={out[25]} pool={out[30]} "
              f"per call cyc: deq {out[26] / w:.0f} reserve {out[27] / w:.0f} claim {out[28] / w:.0f} "
              f"enq {out[29] / w:.0f} total {out[31] / w:.0f}; block_init {out[21] / max(out[20], 1):.0f} "
              f"kernel body {out[22] / max(out[20], 1):.0f}")
        h.launch_free(n, ptrs); torch.cuda.synchronize()
