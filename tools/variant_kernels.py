"""2^20-thread alloc / free launches of one variant (for ncu captures and timing):
python tools/variant_kernels.py <size> <kind> <flavor> <heap GiB> [iters]
Prints per-launch event times of the alloc and free kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

size, kind, flavor = (int(x) for x in sys.argv[1:4])
heap = int(float(sys.argv[4]) * (1 << 30)) if len(sys.argv) > 4 else 1 << 30
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 4
n = 1 << 20
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
hc = ob.HeapConfig(heap, allocator_kind=ob.AllocatorKind(kind), queue_flavor=ob.QueueFlavor(flavor))
with ob.Heap(hc) as h:
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for it in range(iters):
        ev[0].record(); h.launch_alloc(n, ptrs, size=size); ev[1].record()
        ev[2].record(); h.launch_free(n, ptrs); ev[3].record()
        torch.cuda.synchronize()
        print(f"{ob.variant_name(hc.variant)} {size} B: alloc {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us "
              f"free {ev[2].elapsed_time(ev[3]) * 1e3:.1f} us")
    assert h.last_error()[0] == 0
