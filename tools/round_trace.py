"""Where a failed retry round's time goes (experiment build with -DOURO_ROUND_TRACE):
OURO_B200_LIB=exp/lib_trace.so python tools/round_trace.py [size] [kind] [threads]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

size = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 20
L = ob.lib()
buf = (C.c_ulonglong * 8)()
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
with ob.Heap(ob.HeapConfig(1 << 30, allocator_kind=ob.AllocatorKind(kind))) as h:
    for it in range(3):
        L.ouro_debug_trace(buf, 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.launch_alloc(n, ptrs, size=size); b.record(); b.synchronize()
        L.ouro_debug_trace(buf, 1)
        t = list(buf)
        pr = lambda x, y: x / max(y, 1)
        print(f"alloc_us={a.elapsed_time(b) * 1000:.1f} polls={t[1]} count-load cyc/poll={pr(t[0], t[1]):.0f} "
              f"poll_after calls={t[3]} cyc/call={pr(t[2], t[3]):.0f} iters/call={pr(t[6], t[3]):.2f} "
              f"rounds={t[5]} cyc/round={pr(t[4], t[5]):.0f} backoff cyc/round={pr(t[7], t[5]):.0f}")
        h.launch_free(n, ptrs); torch.cuda.synchronize()
