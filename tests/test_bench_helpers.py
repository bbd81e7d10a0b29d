"""bench.py's derived numbers (CPU): the OOM-storm latency roofline and the
algorithmic work per pair that the roofline fractions are computed from."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_storm_roofline_floor_and_selection():
    n = 1 << 20
    per = {"16": {"oom": 0, "alloc_us": 37.0},          # fully served: not a storm
           "128": {"oom": n // 5, "alloc_us": 90.0},    # 20 % OOM: not a storm
           "8192": {"oom": n - 13104, "alloc_us": 236.0}}
    r = bench.storm_roofline(per, n, max_retries=64, hot_lat_s=220e-9, block=256)
    waves = n / (256 * 6 * 148)
    floor = waves * 63 * 220e-9 * 1e6
    assert r["bound"] == "latency" and r["rounds"] == 63
    assert abs(r["waves"] - round(waves, 2)) < 1e-9
    assert set(r["per_size"]) == {"8192"}
    p = r["per_size"]["8192"]
    assert abs(p["floor_us"] - round(floor, 1)) < 1e-9
    assert abs(p["frac"] - round(floor / 236.0, 3)) < 1e-9
    assert 0 < p["frac"] < 1


def test_rmw_per_pair_matches_survey_table():
    # PQ 2.125 element-ops per pair; CQ 16 B 0.315, 1 KiB 0.453, 8 KiB 2.0
    assert abs(bench.rmw_per_pair(0, 0, 16) - 2.125) < 1e-9
    assert abs(bench.rmw_per_pair(1, 0, 16) - 0.315) < 2e-3
    assert abs(bench.rmw_per_pair(1, 0, 1024) - 0.453) < 2e-3
    assert abs(bench.rmw_per_pair(1, 0, 8192) - 2.0) < 2e-3


def test_page_bytes_rounds_to_class():
    assert [bench.page_bytes(s) for s in (4, 16, 17, 1000, 1024, 8192)] == [16, 16, 32, 1024, 1024, 8192]


def test_sweep_floor_mixes_chain_and_storm_floors():
    n = 1 << 20
    per = {"16": {"ok": n, "oom": 0, "alloc_us": 36.0},
           "8192": {"ok": 13104, "oom": n - 13104, "alloc_us": 236.0}}
    r = bench.sweep_floor(per, n, 64, 220e-9, 256, p_same=1.45e9)
    chain16 = (n // 32) / 1.45e9 * 1e6
    storm = bench.storm_roofline(per, n, 64, 220e-9, 256)["per_size"]["8192"]["floor_us"]
    assert abs(r["floor_us"] - round(chain16 + storm, 1)) < 0.2
    assert r["alloc_us"] == 272.0 and 0 < r["frac"] < 1
