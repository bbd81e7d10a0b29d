"""configs[0] timing: 65 536 x malloc(16) / free on the 64 MiB chunk heap, per-launch event times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

n = 65536
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with ob.Heap(ob.HeapConfig(64 << 20, allocator_kind=ob.AllocatorKind.Chunk)) as h:
    a, f = [], []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for it in range(8):
        flush.fill_(it)
        ev[0].record(); h.launch_alloc(n, ptrs, size=16); ev[1].record()
        flush.fill_(it + 1)
        ev[2].record(); h.launch_free(n, ptrs); ev[3].record()
        torch.cuda.synchronize()
        if it >= 3:
            a.append(ev[0].elapsed_time(ev[1]) * 1e3); f.append(ev[2].elapsed_time(ev[3]) * 1e3)
    print(f"{os.environ.get('OURO_B200_LIB', 'tree').split('/')[-1]}: alloc {sorted(a)[len(a)//2]:.1f} us free {sorted(f)[len(f)//2]:.1f} us")
    import ctypes as C
    out = (C.c_uint64 * 32)()
    if hasattr(ob.lib(), "ouro_debug_counters") and ob.lib().ouro_debug_counters(out, 1) == 0 and any(out):
        print("  counters (8 launches):", list(out)[:16])
    st = h.stats()
    print("  pool dequeues / stale drops:", st.stale_drops, "chunks per class:", [st.cls[k].chunks for k in range(3)])
