"""configs[3] page-kind churn with the retry-machinery counters of an OURO_STORM_STATS=1 build:
OURO_B200_LIB=exp_stats/X.so python tools/churn_stats.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

n = 1 << 22
L = ob.lib()
L.ouro_debug_counters.argtypes = [C.POINTER(C.c_uint64), C.c_int]
out = (C.c_uint64 * 32)()
with ob.Heap(ob.HeapConfig(16 << 30, allocator_kind=ob.AllocatorKind(0))) as h:
    slots = torch.zeros(n, dtype=torch.int64, device="cuda")
    res = torch.zeros(5, dtype=torch.int64, device="cuda")
    r0 = 0
    for it in range(4):
        L.ouro_debug_counters(out, 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.launch_churn(n, r0, 10, 1, slots, res); b.record(); b.synchronize()
        r0 += 10
        L.ouro_debug_counters(out, 1)
        print(f"churn-pq 10 rounds {a.elapsed_time(b) * 1000:.0f} us  loops={out[0]} rounds={out[1]} "
              f"observe_once={out[5]} reserve_RMWs={out[7]} pump_rounds={out[14]} "
              f"cyc/round={out[11] / max(out[1], 1):.0f} rounds/loop={out[1] / max(out[0], 1):.2f}")
