"""Repro loop for the chunk-kind double-free accounting test: 65 536 x malloc(48),
free all, free all again; every second free must be DoubleFree or InvalidHandle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_18211_b200 as ob
flavor = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n = 1 << 16
bad = 0
for rep in range(reps):
    hc = ob.HeapConfig(64 << 20, 64 << 10, 16, 8192, ob.QueueFlavor(flavor), ob.AllocatorKind(1),
                       ob.BackoffPolicy(0), 64)
    with ob.Heap(hc) as h:
        ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
        h.launch_alloc(n, ptrs, size=48)
        torch.cuda.synchronize()
        a = h.audit(n, ptrs)
        s0 = h.stats()
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        s1 = h.stats()
        d1 = h.digest()
        h.launch_free(n, ptrs)
        torch.cuda.synchronize()
        s = h.stats()
        first, mask = h.last_error(clear=True)
        tot = s.double_frees + s.invalid_frees
        ok = tot == n
        if not ok:
            bad += 1
        print(f"rep {rep}: live {a.live} overlaps {a.overlaps} | after 1st: dbl {s1.double_frees} inv {s1.invalid_frees} "
              f"live_pages {d1.live_pages} | after 2nd: dbl {s.double_frees} inv {s.invalid_frees} "
              f"sum {tot} {'OK' if ok else 'MISSING %d' % (n - tot)} mask {mask:#x} timeouts {s.timeouts} corr {s.corruptions} stale {s.stale_drops}")
print("bad reps", bad)
