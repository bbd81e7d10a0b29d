"""Sweep driver, CSV emitter and command-line front end.

Follows the reference SPEC's ``bench`` and ``cli`` modules:
  run_sweep   SPEC.md:397-404  (BySize at 1024 allocations / ByCount at 1000 B; one
                                TrialResult per point; a failing point is flagged and
                                the sweep continues)
  emit_csv    SPEC.md:405-409  (header ``variant,axis,point,iteration,alloc_ms,free_ms,
                                mean_all_ms,mean_subsequent_ms,verified``; one row per
                                (point, iteration) plus one summary row per point;
                                deterministic order; RFC-4180 quoting)
  parse_args  SPEC.md:433-447  (trial | sweep | selftest; defaults heap 64 MiB, chunk
                                64 KiB, iterations 10, backoff fence; --iterations 1 is a
                                usage error; OURO_THREADS overrides the --threads default)
  main        SPEC.md:448-452  (exit 0 iff every trial verified, 1 on any trial failure,
                                2 on usage error; CSV on stdout, logs on stderr)

Every trial runs on the GPU through the C-ABI (``ouro_run_trial``: one thread per
allocation, alloc -> write -> verify -> free per iteration, CUDA-event timings), so
``--threads`` is recorded but the launch is always one thread per allocation.

    python -m paper_2504_18211_b200 trial --variant page --allocations 1024 --size-bytes 1000
    python -m paper_2504_18211_b200 sweep --variant vl-chunk --out sweep.csv
    python -m paper_2504_18211_b200 selftest
"""
from __future__ import annotations

import argparse
import csv
import io
import os
import sys
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

HEADER = ["variant", "axis", "point", "iteration", "alloc_ms", "free_ms",
          "mean_all_ms", "mean_subsequent_ms", "verified"]
DEFAULT_SIZE_POINTS = [1000, 2000, 3000, 4000, 5000, 6000, 7000, 8000]   # Fig. 1-6 x-axis
DEFAULT_COUNT_POINTS = [1000, 2000, 3000, 4000, 5000, 6000, 7000, 8000, 9000]
FIXED_COUNT = 1024     # BySize: "as a function of allocation size for 1024 allocations"
FIXED_SIZE = 1000      # ByCount: "for an allocation size of 1000 bytes"
VARIANT_NAMES = ("page", "chunk", "va-page", "va-chunk", "vl-page", "vl-chunk")

EXIT_OK, EXIT_TRIAL_FAILED, EXIT_USAGE = 0, 1, 2


class UsageError(Exception):
    """Bad command line; names the offending flag."""


@dataclass
class PointResult:
    """One TrialResult of a sweep."""
    variant: str
    axis: str                   # "size" | "count"
    point: int
    alloc_ms: List[float] = field(default_factory=list)
    free_ms: List[float] = field(default_factory=list)
    mean_all_ms: Optional[float] = None
    mean_subsequent_ms: Optional[float] = None
    status: str = "pass"        # pass | oom | corrupt | error

    @property
    def ok(self) -> bool:
        return self.status == "pass"


def trial_means(ms: Sequence[float]):
    """mean_all over 1..n, mean_subsequent over 2..n."""
    if len(ms) < 2:
        raise ValueError("iterations >= 2 required (SPEC.md:371)")
    return sum(ms) / len(ms), sum(ms[1:]) / (len(ms) - 1)


# ------------------------------------------------------------------ CSV ----
def _fmt(x: Optional[float]) -> str:
    return "" if x is None else f"{x:.6f}"   # ms with >= microsecond resolution


def emit_csv(table: Sequence[PointResult]) -> str:
    """Rows ordered by (variant, axis, point) then iteration; the summary row of a
    point follows its iterations with iteration = "summary"."""
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\r\n", quoting=csv.QUOTE_MINIMAL)
    w.writerow(HEADER)
    for r in sorted(table, key=lambda r: (r.variant, r.axis, r.point)):
        for i, (a, f) in enumerate(zip(r.alloc_ms, r.free_ms), start=1):
            w.writerow([r.variant, r.axis, r.point, i, _fmt(a), _fmt(f), "", "", r.status])
        w.writerow([r.variant, r.axis, r.point, "summary", "", "",
                    _fmt(r.mean_all_ms), _fmt(r.mean_subsequent_ms), r.status])
    return out.getvalue()


def parse_csv(text: str) -> List[PointResult]:
    """Inverse of emit_csv (the SPEC's parse-back oracle)."""
    rows = list(csv.reader(io.StringIO(text)))
    if not rows or rows[0] != HEADER:
        raise ValueError("not an ouro sweep CSV (header mismatch)")
    table: List[PointResult] = []
    cur: Optional[PointResult] = None
    for row in rows[1:]:
        variant, axis, point, it, a, f, ma, ms, st = row
        key = (variant, axis, int(point))
        if cur is None or (cur.variant, cur.axis, cur.point) != key:
            cur = PointResult(variant, axis, int(point), status=st)
            table.append(cur)
        if it == "summary":
            cur.mean_all_ms = float(ma) if ma else None
            cur.mean_subsequent_ms = float(ms) if ms else None
            cur.status = st
        else:
            cur.alloc_ms.append(float(a))
            cur.free_ms.append(float(f))
    return table


# -------------------------------------------------------------- trials ----
def auto_heap_bytes(kind: int, demand: Sequence[tuple], chunk_bytes: int = 64 << 10,
                    min_page: int = 16, max_page: int = 8192) -> int:
    """run_trial's precondition: the arena fits the demand with >= 2x
    headroom.  demand = [(allocations, bytes)]; the page allocator partitions the heap
    equally over its classes, so it needs classes x the largest class
    demand; the chunk allocator needs whole chunks plus virtual-queue segments."""
    classes = (max_page // min_page).bit_length()
    need = 0
    for n, b in demand:
        pb = max(min_page, 1 << (max(b, 1) - 1).bit_length())
        ppc = max(1, chunk_bytes // pb)
        chunks = -(-n // ppc)
        need = max(need, (classes if kind == 0 else 1) * chunks * chunk_bytes)
    heap = 64 << 20
    while heap < 2 * need + (16 << 20):
        heap *= 2
    return heap


def _heap_config(args, variant: str, demand: Sequence[tuple] = ()):
    import paper_2504_18211_b200 as ob
    v = ob.variant_from_name(variant)
    if v is None:
        raise UsageError(f"--variant: unknown variant {variant!r} (one of {', '.join(VARIANT_NAMES)})")
    heap = args.heap_bytes if args.heap_bytes else auto_heap_bytes(int(v.kind), demand, args.chunk_bytes)
    hc = ob.HeapConfig(heap_bytes=heap, chunk_bytes=args.chunk_bytes,
                       queue_flavor=v.flavor, allocator_kind=v.kind, max_retries=args.max_retries,
                       backoff=ob.BackoffPolicy.SleepRetry if args.backoff == "sleep" else ob.BackoffPolicy.FenceRetry)
    try:
        hc.validate()
    except ob.ConfigError as e:
        raise UsageError(f"--heap-bytes/--chunk-bytes: {e}") from e
    return hc


def run_point(heap, variant: str, axis: str, point: int, n: int, nbytes: int, iterations: int,
              seed: int) -> PointResult:
    """One trial; OOM is a failed result, not a crash."""
    r = PointResult(variant, axis, point)
    try:
        t = heap.run_trial(n, nbytes, iterations=iterations, seed=seed)
    except Exception as e:  # noqa: BLE001 - reported per point, the sweep continues
        print(f"ouro: {variant} {axis}={point}: {e}", file=sys.stderr)
        r.status = "error"
        return r
    r.alloc_ms = [t.alloc_ms[i] for i in range(t.iterations)]
    r.free_ms = [t.free_ms[i] for i in range(t.iterations)]
    r.mean_all_ms, r.mean_subsequent_ms = t.mean_all_ms, t.mean_subsequent_ms
    if not t.verified:
        r.status = "corrupt"
    elif t.failed_allocs:
        r.status = "oom"
    return r


def run_sweep(heap, variant: str, axis: str, points: Sequence[int], fixed: int, iterations: int,
              seed: int) -> List[PointResult]:
    """BySize: `fixed` allocations over sizes; ByCount: `fixed` bytes over counts."""
    if not points or list(points) != sorted(points):
        raise UsageError("--points: must be nonempty and ascending (SPEC.md:399)")
    out = []
    for p in points:
        n, nbytes = (fixed, p) if axis == "size" else (p, fixed)
        out.append(run_point(heap, variant, axis, p, n, nbytes, iterations, seed))
    return out


def selftest(args) -> List[PointResult]:
    """Acceptance criteria 1, 2 and 8 on all six variants: 1024
    allocations x {16, 1000, 1024, 8192} B x 10 iterations verify clean with no leaked
    page (digest at quiescence: live = 0, partition intact); the statistics contract;
    an over-capacity trial fails without aborting and a normal trial passes after it."""
    import paper_2504_18211_b200 as ob
    a, s = trial_means([10, 1, 1, 1, 1, 1, 1, 1, 1, 1])
    if abs(a - 1.9) > 1e-12 or s != 1.0:
        raise AssertionError("statistics contract (criterion 2) violated")
    table = []
    for name in VARIANT_NAMES:
        hc = _heap_config(args, name, [(1024, 8192)])
        with ob.Heap(hc) as h:
            for size in (16, 1000, 1024, 8192):
                r = run_point(h, name, "size", size, 1024, size, 10, args.seed)
                d = h.digest()
                if r.ok and (d.live_pages != 0 or d.partition_ok != 1 or h.last_error()[0] != 0):
                    r.status = "corrupt"
                table.append(r)
            cap = hc.heap_bytes // 8192 + 1024          # more 8 KiB pages than the heap holds
            r = run_point(h, name, "count", cap, cap, 8192, 2, args.seed)
            oom_ok = r.status == "oom"
            r2 = run_point(h, name, "count", 1024, 1024, 1000, 2, args.seed)
            if not oom_ok or not r2.ok:
                r2.status = "error"
                print(f"ouro: selftest {name}: OOM resilience failed ({r.status}, {r2.status})",
                      file=sys.stderr)
            table.append(r2)
    return table


# ----------------------------------------------------------------- CLI ----
class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors -> UsageError (exit 2), not SystemExit
        raise UsageError(message)


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="python -m paper_2504_18211_b200", description="Ouroboros B200 allocator driver")
    p.add_argument("command", choices=["trial", "sweep", "selftest"])
    p.add_argument("--max-retries", type=int, default=64)
    p.add_argument("--variant", default="page", choices=VARIANT_NAMES)
    p.add_argument("--heap-bytes", type=int, default=0,
                   help="0 (default): 64 MiB, grown to fit the demand with 2x headroom (SPEC.md:380)")
    p.add_argument("--chunk-bytes", type=int, default=64 << 10)
    p.add_argument("--allocations", type=int, default=FIXED_COUNT)
    p.add_argument("--size-bytes", type=int, default=FIXED_SIZE)
    p.add_argument("--iterations", type=int, default=10)
    p.add_argument("--threads", type=int, default=None,
                   help="recorded only: the GPU launches one thread per allocation (env OURO_THREADS)")
    p.add_argument("--backoff", default="fence", choices=["fence", "sleep"])
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--axis", default="size", choices=["size", "count"], help="sweep axis (BySize/ByCount)")
    p.add_argument("--points", default=None, help="comma-separated ascending sweep points")
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--out", default="-", help="CSV path, '-' = stdout")
    return p


def parse_args(argv: Sequence[str]):
    a = build_parser().parse_args(list(argv))
    if a.iterations < 2:
        raise UsageError("--iterations: must be >= 2 (the subsequent mean needs two, SPEC.md:371)")
    if a.iterations > 64:
        raise UsageError("--iterations: at most 64")
    if a.allocations < 1:
        raise UsageError("--allocations: must be >= 1")
    if a.size_bytes < 1:
        raise UsageError("--size-bytes: must be >= 1")
    if a.threads is None and os.environ.get("OURO_THREADS"):
        try:
            a.threads = int(os.environ["OURO_THREADS"])
        except ValueError as e:
            raise UsageError("OURO_THREADS: not an integer") from e
    if a.threads is not None and a.threads < 1:
        raise UsageError("--threads: must be >= 1")
    if a.points is not None:
        try:
            a.points = [int(x) for x in a.points.split(",") if x.strip()]
        except ValueError as e:
            raise UsageError("--points: comma-separated integers expected") from e
        if not a.points or a.points != sorted(a.points) or a.points[0] < 1:
            raise UsageError("--points: must be nonempty, positive and ascending (SPEC.md:399)")
    return a


def main(argv: Optional[Sequence[str]] = None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    try:
        args = parse_args(argv)
        if args.command == "trial":
            hc = _heap_config(args, args.variant, [(args.allocations, args.size_bytes)])
        elif args.command == "sweep":
            if args.axis == "size":
                demand = [(args.allocations, p) for p in (args.points or DEFAULT_SIZE_POINTS)]
            else:
                demand = [(p, args.size_bytes) for p in (args.points or DEFAULT_COUNT_POINTS)]
            hc = _heap_config(args, args.variant, demand)
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    import paper_2504_18211_b200 as ob
    try:
        if args.command == "selftest":
            table = selftest(args)
        else:
            with ob.Heap(hc, device=args.device) as h:
                if args.command == "trial":
                    table = [run_point(h, args.variant, "size", args.size_bytes, args.allocations,
                                       args.size_bytes, args.iterations, args.seed)]
                else:
                    if args.axis == "size":
                        pts, fixed = args.points or DEFAULT_SIZE_POINTS, args.allocations
                    else:
                        pts, fixed = args.points or DEFAULT_COUNT_POINTS, args.size_bytes
                    table = run_sweep(h, args.variant, args.axis, pts, fixed, args.iterations, args.seed)
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    text = emit_csv(table)
    if args.out == "-":
        sys.stdout.write(text)
        sys.stdout.flush()
    else:
        with open(args.out, "w", newline="") as f:
            f.write(text)
    bad = [r for r in table if not r.ok]
    for r in bad:
        print(f"ouro: {r.variant} {r.axis}={r.point}: {r.status}", file=sys.stderr)
    return EXIT_OK if not bad else EXIT_TRIAL_FAILED


if __name__ == "__main__":
    sys.exit(main())
