"""VLPQ 8 GiB, 2^20 x malloc(16) / free cycles: per-launch times, for ncu captures
(ncu -k regex:k_alloc -s 3 -c 1 ... python tools/vl_probe.py)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_18211_b200 as ob
flavor = int(sys.argv[1]) if len(sys.argv) > 1 else 2
size = int(sys.argv[2]) if len(sys.argv) > 2 else 16
n = 1 << 20
ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
hc = ob.HeapConfig(8 << 30, queue_flavor=ob.QueueFlavor(flavor))
with ob.Heap(hc) as h:
    ring = h.vl_ring(0)
    c, hd, vh, vt = h.queue_links(0)
    print("init: head", vh >> 32, "tail", vt >> 32, "ring", [(x >> 32, x & 0xffffffff) for x in ring[:3]], [(x >> 32) for x in ring[250:256]])
    for it in range(5):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(); h.launch_alloc(n, ptrs, size=size); ev[1].record()
        h.launch_free(n, ptrs); ev[2].record(); ev[2].synchronize()
        s = h.stats()
        c, hd, vh, vt = h.queue_links(0)
        ring = h.vl_ring(0)
        hs = vh >> 32
        cover = sum(1 for x in range(hs, hs + 256) if ring[x % 256] >> 32 == x and ring[x % 256] != 2**64 - 1)
        print(f"      count {c} head {hd} vl_head seq {hs} vl_tail seq {vt >> 32} ring covers {cover}/256 ahead")
        print(f"it {it}: alloc {ev[0].elapsed_time(ev[1])*1e3:.1f} us free {ev[1].elapsed_time(ev[2])*1e3:.1f} us "
              f"seg_live {s.cls[0].seg_live} hwm {s.cls[0].seg_hwm} err {h.last_error()[0]}")
