"""Logical reference model (free-list / bitset form) of the single-lane allocator
protocol -- SPEC.md acceptance criterion 3 ("matches a reference free-list/bitset
oracle on success/failure of every op").  Pure Python, small heaps only.

It is a second, independent restatement of DESIGN.md §3: per-class FIFO
free-lists for the page kind, and for the chunk kind a
FIFO pool, per-class FIFO chunk queues, Python-int bitsets, the in-transit rule
(SPEC.md:299), 0->1 re-enqueue (227), watermark return-to-pool (228, gap G3) and
virtual-queue segment traffic.  The C oracle must agree
with it offset-for-offset on every op.
"""
from collections import deque

OK, INVALID, DOUBLE_FREE, OOM, TOO_LARGE = 0, 2, 3, 7, 8


def _log2(x):
    return x.bit_length() - 1


class Model:
    def __init__(self, heap, chunk, minp, maxp, kind, flavor, max_retries=64):
        self.heap, self.chunk, self.minp, self.maxp = heap, chunk, minp, maxp
        self.kind, self.flavor, self.max_retries = kind, flavor, max_retries
        self.N = heap // chunk
        self.K = _log2(maxp // minp) + 1
        self.page_bits = _log2(chunk // minp)
        self.chunk_bits = (self.N - 1).bit_length()
        self.gmask = (1 << min(24, 32 - self.chunk_bits)) - 1
        self.S_va = chunk // 8
        self.S_vl = chunk // 8 - 2
        self.state = [0] * self.N
        self.free = [0] * self.N
        self.gen = [0] * self.N
        self.bits = [0] * self.N
        if kind == 0:
            self._build_page()
        else:
            self._build_chunk()

    def ppc(self, k):
        return self.chunk // (self.minp << k)

    def page_bytes(self, k):
        return self.minp << k

    def off(self, c, k, p):
        return c * self.chunk + p * self.page_bytes(k)

    # ------------------------------------------------------------ page kind
    def _build_page(self):
        N, K = self.N, self.K
        self.q = []
        start = 0
        for k in range(K):
            n = N // K + (N % K if k == 0 else 0)
            s = 0
            if self.flavor != 0:
                S = self.S_va if self.flavor == 1 else self.S_vl
                for s in range(n + 1):
                    cap = (n - s) * self.ppc(k)
                    need = 0 if cap == 0 else -(-cap // S) + 2
                    if need <= s:
                        break
            dq = deque()
            for i in range(n):
                c = start + i
                if i < s:
                    self.state[c] = 0xFF
                else:
                    self.state[c] = k + 1
                    self.free[c] = self.ppc(k)
                    self.gen[c] = 1
                    self.bits[c] = (1 << self.ppc(k)) - 1
                    for p in range(self.ppc(k)):
                        dq.append((c, p))
            self.q.append(dq)
            start += n

    # ----------------------------------------------------------- chunk kind
    def _build_chunk(self):
        self.pool = deque(range(self.N))
        self.cq = [deque() for _ in range(self.K)]
        self.assigned = [0] * self.K
        self.floor = 0 if self.flavor == 0 else min(self.K, self.N // 8)
        # virtual-queue bookkeeping per class queue
        self.tail = [0] * self.K
        self.head = [0] * self.K
        self.segs = [dict() for _ in range(self.K)]  # seq -> [chunk, counter]

    def _S(self):
        return self.S_va if self.flavor == 1 else self.S_vl

    def _seg_create(self, k, s):
        c = self.pool.popleft()  # segment supply ignores the floor
        self.segs[k][s] = [c, 0]
        if self.flavor == 2 and s > 0:
            self._vl_add(k, s - 1, 1)

    def _vl_add(self, k, s, n):
        self.segs[k][s][1] += n
        # advance over complete head segments, in order
        while self.segs[k]:
            h = min(self.segs[k])
            if self.segs[k][h][1] != self.S_vl + 1:
                break
            self.pool.append(self.segs[k].pop(h)[0])

    def _enq(self, k, e):
        if self.flavor != 0:
            t = self.tail[k]
            if t % self._S() == 0:
                self._seg_create(k, t // self._S())
        self.tail[k] += 1
        self.cq[k].append(e)

    def _deq(self, k):
        e = self.cq[k].popleft()
        t = self.head[k]
        self.head[k] += 1
        if self.flavor == 1:
            s = t // self.S_va
            self.segs[k][s][1] += 1
            if self.segs[k][s][1] == self.S_va:
                self.pool.append(self.segs[k].pop(s)[0])
        elif self.flavor == 2:
            self._vl_add(k, t // self.S_vl, 1)
        return e

    def _entry(self, c, g):
        return c | ((g & self.gmask) << self.chunk_bits)

    # ------------------------------------------------------------------ ops
    def size_class(self, req):
        if req == 0 or req > self.maxp:
            return None
        lg = 0 if req <= 1 else (req - 1).bit_length()
        ms = _log2(self.minp)
        return lg - ms if lg > ms else 0

    def alloc(self, req):
        k = self.size_class(req)
        if k is None:
            return None, TOO_LARGE
        if self.kind == 0:
            if self.q[k]:
                c, p = self.q[k].popleft()
                self.bits[c] &= ~(1 << p)
                self.free[c] -= 1
                return self.off(c, k, p), OK
            return None, OOM
        attempt = 0
        while True:
            if self.cq[k]:
                e = self._deq(k)
                c = e & ((1 << self.chunk_bits) - 1)
                glow = e >> self.chunk_bits
                if self.state[c] != k + 1 or (self.gen[c] & self.gmask) != glow or self.free[c] == 0:
                    continue
                old = self.free[c]
                self.free[c] -= 1
                b = self.bits[c]
                p = (b & -b).bit_length() - 1
                self.bits[c] &= ~(1 << p)
                if old - 1 > 0:
                    self._enq(k, e)
                return self.off(c, k, p), OK
            if len(self.pool) - self.floor > 0:
                c = self.pool.popleft()
                assert self.state[c] == 0
                self.gen[c] = (self.gen[c] + 1) & 0xFFFFFF
                self.state[c] = k + 1
                ppc = self.ppc(k)
                self.bits[c] = ((1 << ppc) - 1) & ~1
                self.free[c] = ppc - 1
                self.assigned[k] += 1
                if ppc - 1 > 0:
                    self._enq(k, self._entry(c, self.gen[c]))
                return self.off(c, k, 0), OK
            attempt += 1
            if attempt >= self.max_retries:
                return None, OOM

    def dealloc(self, off):
        if off >= self.heap:
            return INVALID
        c = off // self.chunk
        st = self.state[c]
        if st == 0 or st == 0xFF or st > self.K:
            return INVALID
        k = st - 1
        inner = off % self.chunk
        if inner % self.page_bytes(k):
            return INVALID
        p = inner // self.page_bytes(k)
        if (self.bits[c] >> p) & 1:
            return DOUBLE_FREE
        self.bits[c] |= 1 << p
        old = self.free[c]
        self.free[c] += 1
        if self.kind == 0:
            self.q[k].append((c, p))
            return OK
        closed = False
        if self.free[c] == self.ppc(k) and self.assigned[k] > 1:
            self.assigned[k] -= 1
            self.state[c] = 0
            self.free[c] = 0
            self.bits[c] = 0
            self.pool.append(c)
            closed = True
        if not closed and old == 0:
            self._enq(k, self._entry(c, self.gen[c]))
        return OK
