"""Sweep driver, CSV emitter and CLI.  CPU tests cover argument
validation, the exit-code contract for usage errors and the CSV format/parse-back;
GPU tests run trials, sweeps and the selftest through the C-ABI."""
import subprocess
import sys

import pytest

from paper_2504_18211_b200 import cli

ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))


def _run(*argv, env=None):
    return subprocess.run([sys.executable, "-m", "paper_2504_18211_b200", *argv], cwd=ROOT,
                          capture_output=True, text=True, env=env, timeout=600)


# ------------------------------------------------------------------ CSV ----
def test_csv_empty_table_is_header_only():
    """empty table -> header only."""
    assert cli.emit_csv([]) == ",".join(cli.HEADER) + "\r\n"


def test_csv_two_iterations_two_detail_rows_one_summary():
    """one trial, 2 iterations -> 2 detail + 1 summary row."""
    r = cli.PointResult("page", "size", 1000, [0.5, 0.25], [0.125, 0.0625], *cli.trial_means([0.5, 0.25]))
    lines = cli.emit_csv([r]).split("\r\n")
    assert lines[-1] == "" and len(lines) == 5
    assert lines[1].split(",")[:6] == ["page", "size", "1000", "1", "0.500000", "0.125000"]
    assert lines[2].split(",")[3] == "2"
    s = lines[3].split(",")
    assert s[3] == "summary" and float(s[6]) == 0.375 and float(s[7]) == 0.25 and s[8] == "pass"


def test_csv_round_trip_and_quoting():
    """round-trip parse of emitted CSV reproduces the table; RFC-4180 quoting."""
    t = [cli.PointResult("vl-chunk", "count", 9000, [1.0, 2.0, 3.0], [0.5, 0.5, 0.5], 2.0, 2.5, "pass"),
         cli.PointResult("page", "size", 8000, [4.0, 4.0], [1.0, 1.0], 4.0, 4.0, "oom"),
         cli.PointResult('odd,"name"', "size", 16, [0.001, 0.002], [0.003, 0.004], 0.0015, 0.002, "pass")]
    text = cli.emit_csv(t)
    assert '"odd,""name"""' in text
    back = cli.parse_csv(text)
    key = lambda r: (r.variant, r.axis, r.point)
    for a, b in zip(sorted(t, key=key), back):
        assert (a.variant, a.axis, a.point, a.status) == (b.variant, b.axis, b.point, b.status)
        assert a.alloc_ms == pytest.approx(b.alloc_ms, abs=1e-6) and a.free_ms == pytest.approx(b.free_ms, abs=1e-6)
        assert a.mean_all_ms == pytest.approx(b.mean_all_ms) and a.mean_subsequent_ms == pytest.approx(b.mean_subsequent_ms)


def test_csv_deterministic_order():
    t = [cli.PointResult("page", "size", p, [1.0, 1.0], [1.0, 1.0], 1.0, 1.0) for p in (3000, 1000, 2000)]
    pts = [int(l.split(",")[2]) for l in cli.emit_csv(t).split("\r\n")[1:] if l]
    assert pts == sorted(pts)


def test_statistics_contract():
    """Acceptance criterion 2."""
    a, s = cli.trial_means([10, 1, 1, 1, 1, 1, 1, 1, 1, 1])
    assert a == pytest.approx(1.9) and s == 1.0


# ---------------------------------------------------------------- usage ----
def test_parse_defaults():
    """`trial --variant page --allocations 1024 --size-bytes 1000` -> defaults filled."""
    a = cli.parse_args(["trial", "--variant", "page", "--allocations", "1024", "--size-bytes", "1000"])
    assert (a.heap_bytes, a.chunk_bytes, a.iterations, a.backoff) == (0, 64 << 10, 10, "fence")
    assert cli.auto_heap_bytes(0, [(1024, 1000)]) == 64 << 20          # the SPEC default when it fits
    assert cli.auto_heap_bytes(0, [(1024, 8192)]) == 256 << 20         # page partition: 10 classes x 2x
    b = cli.parse_args(["sweep", "--variant", "vl-chunk"])
    assert b.axis == "size" and b.points is None


@pytest.mark.parametrize("argv", [
    ["trial", "--iterations", "1"],
    ["trial", "--bogus"],                            # bad flag
    ["frobnicate"],                                  # bad subcommand
    ["trial", "--variant", "heap"],                  # unknown variant
    ["trial", "--chunk-bytes", "3072"],              # HeapConfig invariant (power of two)
    ["sweep", "--points", "3000,1000"],              # points not ascending
])
def test_usage_errors_exit_2(argv):
    r = _run(*argv)
    assert r.returncode == 2, (r.stdout, r.stderr)
    assert r.stdout == "" and "usage error" in r.stderr


def test_ouro_threads_env():
    import os
    env = dict(os.environ, OURO_THREADS="7")
    os.environ["OURO_THREADS"] = "7"
    try:
        assert cli.parse_args(["trial"]).threads == 7
        assert cli.parse_args(["trial", "--threads", "3"]).threads == 3
    finally:
        del os.environ["OURO_THREADS"]
    env["OURO_THREADS"] = "x"
    assert _run("trial", env=env).returncode == 2


# ------------------------------------------------------------------ GPU ----
@pytest.mark.gpu
def test_trial_exit_0_csv_on_stdout(cuda):
    r = _run("trial", "--variant", "page", "--allocations", "1024", "--size-bytes", "1000")
    assert r.returncode == 0, r.stderr
    t = cli.parse_csv(r.stdout)
    assert len(t) == 1 and t[0].status == "pass" and len(t[0].alloc_ms) == 10
    assert t[0].mean_subsequent_ms == pytest.approx(sum(t[0].alloc_ms[1:]) / 9, abs=2e-6)


@pytest.mark.gpu
def test_trial_oom_exit_1(cuda):
    """trial with OOM-sized demand -> exit 1 (recorded, not a crash)."""
    r = _run("trial", "--variant", "chunk", "--allocations", "20000", "--size-bytes", "8192",
             "--iterations", "2", "--heap-bytes", str(64 << 20))
    assert r.returncode == 1, r.stderr
    assert cli.parse_csv(r.stdout)[0].status == "oom"


@pytest.mark.gpu
def test_sweep_by_count_single_point(cuda, tmp_path):
    """ByCount, single point {1} -> 1 row (+ its iterations)."""
    out = tmp_path / "s.csv"
    r = _run("sweep", "--variant", "va-chunk", "--axis", "count", "--points", "1", "--iterations", "2",
             "--out", str(out))
    assert r.returncode == 0, r.stderr
    t = cli.parse_csv(out.read_text())
    assert [(x.axis, x.point, x.status) for x in t] == [("count", 1, "pass")]


@pytest.mark.gpu
def test_sweep_oom_point_flagged_neighbours_intact(cuda):
    """a sweep with one OOM point flags that row, neighbours intact."""
    # page kind, 256 MiB: the 8 KiB class owns 1/10 of the heap (~3200 pages)
    r = _run("sweep", "--variant", "page", "--axis", "count", "--points", "1000,2000,9000",
             "--size-bytes", "8192", "--heap-bytes", str(256 << 20), "--iterations", "2")
    t = {x.point: x.status for x in cli.parse_csv(r.stdout)}
    assert t == {1000: "pass", 2000: "pass", 9000: "oom"}
    assert r.returncode == 1


@pytest.mark.gpu
def test_default_size_sweep_all_variants(cuda):
    """BySize over {1000..8000 step 1000} -> 8 points, Figure 1's x-axis."""
    for v in cli.VARIANT_NAMES:
        r = _run("sweep", "--variant", v, "--iterations", "3")
        t = cli.parse_csv(r.stdout)
        assert [x.point for x in t] == cli.DEFAULT_SIZE_POINTS and r.returncode == 0, (v, r.stderr)


@pytest.mark.gpu
def test_selftest_exit_0(cuda):
    """selftest runs the invariant suite on all six variants, exit 0."""
    r = _run("selftest")
    assert r.returncode == 0, r.stderr
    t = cli.parse_csv(r.stdout)
    assert len(t) == 6 * 5 and all(x.ok for x in t)
