"""One write + verify pass over 2^20 slots (for ncu captures of k_pattern):
python tools/pattern_run.py <kind> <size>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_18211_b200 as ob

kind, size = int(sys.argv[1]), int(sys.argv[2])
n = 1 << 20
with ob.Heap(ob.HeapConfig(1 << 30, allocator_kind=ob.AllocatorKind(kind))) as h:
    ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
    h.launch_alloc(n, ptrs, size=size)
    res = torch.tensor([0, -1], dtype=torch.int64, device="cuda")
    h.launch_write(n, ptrs, 3, 1)
    h.launch_verify(n, ptrs, 3, 1, res)
    torch.cuda.synchronize()
    live = int((ptrs != 0).sum())
    print(f"kind {kind} size {size} live {live} bytes {live * max(16, 1 << (size - 1).bit_length())} bad {int(res[0])}")
    h.launch_free(n, ptrs)
    torch.cuda.synchronize()
