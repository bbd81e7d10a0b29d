"""OOM storm with the retry-machinery counters of an OURO_STORM_STATS=1 build:
OURO_B200_LIB=exp/lib_stats.so python tools/storm_stats.py [size] [kind]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

NAMES = ["round loops", "rounds", "-", "-", "-", "observe_once", "-", "reserve RMWs", "-", "-", "-",
         "round-loop cycles", "-", "-", "pump rounds"]
size = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = 1 << 20
L = ob.lib()
L.ouro_debug_counters.argtypes = [C.POINTER(C.c_uint64), C.c_int]
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
out = (C.c_uint64 * 32)()
with ob.Heap(ob.HeapConfig(1 << 30, allocator_kind=ob.AllocatorKind(kind))) as h:
    for it in range(3):
        L.ouro_debug_counters(out, 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.launch_alloc(n, ptrs, size=size); b.record(); b.synchronize()
        L.ouro_debug_counters(out, 1)
        print(f"size {size} kind {kind} alloc_us={a.elapsed_time(b) * 1000:.1f}  " +
              "  ".join(f"{nm}={out[i]}" for i, nm in enumerate(NAMES) if nm != "-"))
        if out[1]:
            print(f"   cycles/round {out[11] / out[1]:.0f}  rounds/loop {out[1] / max(out[0], 1):.1f}  "
                  f"pump share of rounds {out[14] / out[1]:.3f}")
        if out[16]:
            print(f"   per OOM warp: pq_alloc->rounds {out[17] / out[16]:.0f} cyc, rounds {out[18] / out[16]:.0f} cyc, "
                  f"after {out[19] / out[16]:.0f} cyc;  per warp: block_init {out[21] / out[20]:.0f} cyc, "
                  f"kernel body {out[22] / out[20]:.0f} cyc ({out[20]} warps)")
        h.launch_free(n, ptrs); torch.cuda.synchronize()
