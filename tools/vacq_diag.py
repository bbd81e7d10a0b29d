"""VACQ 8 GiB sweep: per-class chunks / segments / pool after the 8 KiB alloc phase, GPU vs oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch

import paper_2504_18211_b200 as ob
from oracle_lib import OHeap

kind, flavor = int(sys.argv[1]) if len(sys.argv) > 1 else 1, int(sys.argv[2]) if len(sys.argv) > 2 else 1
hc = ob.HeapConfig(8 << 30, allocator_kind=ob.AllocatorKind(kind), queue_flavor=ob.QueueFlavor(flavor))
n = 1 << 20
oh = OHeap(hc.to_c())
sizes = [16, 32, 64, 128, 256, 512, 1000, 1024, 2048, 4096, 8192]
with ob.Heap(hc) as h:
    ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for s in sizes:
        offs, want = oh.alloc_slots(n, s)
        cnt.zero_()
        h.launch_alloc(n, ptrs, size=s)
        h.launch_count(n, ptrs, cnt)
        torch.cuda.synchronize()
        if s == sizes[-1]:
            gs, os_ = h.stats(), oh.stats()
            print("size", s, "gpu ok", int(cnt), "oracle ok", want)
            print("pool_len gpu", gs.pool_len, "oracle", os_.pool_len, " stale", gs.stale_drops, os_.stale_drops)
            for k in range(gs.num_classes):
                g, o = gs.cls[k], os_.cls[k]
                print(f"  class {k}: chunks {g.chunks}/{o.chunks} live {g.live_pages}/{o.live_pages} "
                      f"qlen {g.queue_len}/{o.queue_len} seg_live {g.seg_live}/{o.seg_live} hwm {g.seg_hwm}/{o.seg_hwm} "
                      f"ooms {g.ooms}/{o.ooms}")
        oh.free_slots(offs)
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        gd, od = h.digest().as_dict(), oh.digest().as_dict()
        if gd != od:
            print("digest differs after", s, {k: (gd[k], od[k]) for k in gd if gd[k] != od[k]})
    print("last error", h.last_error())
