"""Block-fetch counters of an OURO_STORM_STATS=1 build (cq_alloc_block):
OURO_B200_LIB=exp_stats/blkstats.so python tools/blk_stats.py [size] [flavor]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

size = int(sys.argv[1]) if len(sys.argv) > 1 else 16
fl = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = 1 << 20
L = ob.lib()
L.ouro_debug_counters.argtypes = [C.POINTER(C.c_uint64), C.c_int]
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
out = (C.c_uint64 * 32)()
with ob.Heap(ob.HeapConfig(1 << 30, allocator_kind=ob.AllocatorKind(1), queue_flavor=ob.QueueFlavor(fl))) as h:
    for it in range(3):
        L.ouro_debug_counters(out, 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.launch_alloc(n, ptrs, size=size); b.record(); b.synchronize()
        L.ouro_debug_counters(out, 1)
        calls = max(out[2], 1)
        fetches = out[25] + out[28]
        print(f"size {size} alloc_us={a.elapsed_time(b) * 1000:.1f} calls={out[2]} fetch(deq)={out[25]} "
              f"fetch(pool)={out[28]} warps/fetch={out[26] / max(fetches, 1):.2f} short={out[27]} "
              f"became-fetcher={out[29]} wait cyc/call={out[30] / calls:.0f} total cyc/call={out[31] / calls:.0f} "
              f"kernel body {out[22] / max(out[20], 1):.0f}")
        h.launch_free(n, ptrs); torch.cuda.synchronize()
