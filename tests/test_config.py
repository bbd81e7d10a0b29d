"""Config / arena arithmetic: product (libouro_b200 host half), oracle and the
reference's own config.cpp must agree exactly (CPU only, no GPU).

Pins: /root/reference/proj/src/config.cpp:16-59, config.hpp:26-73.
"""
import ctypes as C
import json
import os
import random

import pytest

import paper_2504_18211_b200 as ob
from paper_2504_18211_b200._abi import Config, Geometry
from oracle_lib import oracle, ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _validate(fn, cfg):
    buf = C.create_string_buffer(256)
    st = fn(C.byref(cfg), buf, 256)
    return st, buf.value.decode()


def test_layout_matches_reference():
    v = _load("variants.json")
    lay = v["layout"]
    assert C.sizeof(Config) == lay[0] == 48
    assert C.alignment(Config) == lay[1] == 8
    assert [Config.queue_flavor.offset, Config.allocator_kind.offset, Config.backoff.offset,
            Config.max_retries.offset, Config.sleep_base_ns.offset, Config.sleep_cap_ns.offset] == lay[2:8]


def test_defaults_match_reference():
    v = _load("variants.json")["defaults"]
    c = Config()
    assert ob.lib().ouro_config_default(C.byref(c)) == 0
    got = [c.heap_bytes, c.chunk_bytes, c.min_page_bytes, c.max_page_bytes, c.queue_flavor,
           c.allocator_kind, c.backoff, c.max_retries, c.sleep_base_ns, c.sleep_cap_ns]
    assert got == v
    h = ob.HeapConfig()
    assert [h.heap_bytes, h.chunk_bytes, h.min_page_bytes, h.max_page_bytes, int(h.queue_flavor),
            int(h.allocator_kind), int(h.backoff), h.max_retries, h.sleep_base_ns, h.sleep_cap_ns] == v


def test_validate_golden_grid():
    """Every row of the reference-generated grid: same verdict, same message."""
    g = _load("config_validate.json")
    msgs = g["messages"]
    L, O = ob.lib(), oracle()
    for heap, chunk, mn, mx, retries, valid, mi, nch, mppc in g["rows"]:
        cfg = Config(heap, chunk, mn, mx, 0, 0, 0, 0, retries, 100, 100000)
        for fn in (L.ouro_config_validate, O.orc_config_validate):
            st, msg = _validate(fn, cfg)
            assert (st == 0) == bool(valid), (heap, chunk, mn, mx, retries)
            assert msg == msgs[mi]
        hc = ob.HeapConfig(heap, chunk, mn, mx, max_retries=retries)
        if chunk:
            assert hc.num_chunks() == nch
        if mn:
            assert hc.max_pages_per_chunk() == mppc


def test_validate_live_reference_random():
    R = ref()
    if R is None:
        pytest.skip("reference build unavailable (only the golden grid applies)")
    rng = random.Random(7)
    L = ob.lib()
    for _ in range(3000):
        vals = [rng.choice([1 << rng.randrange(0, 50), rng.randrange(1, 1 << 40)]) for _ in range(4)]
        cfg = Config(*vals, 0, 0, 0, 0, rng.choice([0, 1, 9]), 100, 100000)
        assert _validate(R.ref_validate, cfg) == _validate(L.ouro_config_validate, cfg)


def test_variants_match_reference():
    v = _load("variants.json")["all_variants"]
    assert [(x["kind"], x["flavor"]) for x in v] == [(int(a.kind), int(a.flavor)) for a in ob.ALL_VARIANTS]
    O = oracle()
    for x in v:
        var = ob.Variant(ob.AllocatorKind(x["kind"]), ob.QueueFlavor(x["flavor"]))
        assert ob.variant_name(var) == x["name"]
        assert O.orc_variant_name(x["kind"], x["flavor"]).decode() == x["name"]
        assert ob.variant_from_name(x["name"]) == var
    assert ob.variant_from_name("nope") is None
    assert ob.variant_from_name("PAGE") is None


def test_geometry_kats():
    for row in _load("spec_kats.json")["geometry"]:
        hc = ob.HeapConfig(row["heap"], row["chunk"], row["min"], row["max"])
        if row.get("config_error"):
            with pytest.raises(ob.ConfigError):
                hc.validate()
            continue
        hc.validate()
        g = hc.geometry()
        assert g.num_chunks == row["num_chunks"] and g.num_classes == row["num_classes"]
        og = Geometry()
        assert oracle().orc_config_geometry(C.byref(hc.to_c()), C.byref(og)) == 0
        assert bytes(og) == bytes(g)


def _ref_class(req, minp=16):
    if req == 0 or req > 8192:
        return None
    p = minp
    k = 0
    while p < req:
        p <<= 1
        k += 1
    return k


def test_size_class_exhaustive():
    cfgp = ob.HeapConfig()
    c = cfgp.to_c()
    L, O = ob.lib(), oracle()
    for req in list(range(0, 8200)) + [1 << 20, 1 << 40, 2 ** 64 - 1]:
        want = _ref_class(req)
        for fn in (L.ouro_size_class, O.orc_size_class):
            k = C.c_uint32()
            st = fn(C.byref(c), req, C.byref(k))
            if want is None:
                assert st == ob._abi.ERR_TOO_LARGE
            else:
                assert st == 0 and k.value == want, req
    for row in _load("spec_kats.json")["size_class"]:
        if row.get("too_large"):
            with pytest.raises(ob.OuroError):
                ob.size_class(cfgp, row["req"])
        elif "page_bytes" in row:
            assert 16 << ob.size_class(cfgp, row["req"]) == row["page_bytes"]
        else:
            assert ob.size_class(cfgp, row["req"]) == row["class"]


def test_size_class_monotone_idempotent():
    cfgp = ob.HeapConfig()
    prev = 0
    for req in range(1, 8193):
        k = ob.size_class(cfgp, req)
        assert k >= prev
        prev = k
        assert ob.size_class(cfgp, 16 << k) == k


def test_handles_kats_and_fuzz():
    hc = ob.HeapConfig(1 << 30)
    c = hc.to_c()
    L, O = ob.lib(), oracle()
    for row in _load("spec_kats.json")["handles"]:
        for fn in (L.ouro_handle_encode, O.orc_handle_encode):
            h = C.c_uint32()
            assert fn(C.byref(c), row["chunk"], row["page"], C.byref(h)) == 0
            assert h.value == row["handle"]
    rng = random.Random(11)
    n, ppc = hc.num_chunks(), hc.max_pages_per_chunk()
    for _ in range(100_000 // 4):
        ch, pg = rng.randrange(n), rng.randrange(ppc)
        h = C.c_uint32()
        assert L.ouro_handle_encode(C.byref(c), ch, pg, C.byref(h)) == 0
        assert h.value == (ch << 12) | pg
        a, b = C.c_uint32(), C.c_uint32()
        assert O.orc_handle_decode(C.byref(c), h.value, C.byref(a), C.byref(b)) == 0
        assert (a.value, b.value) == (ch, pg)
    h = C.c_uint32()
    assert L.ouro_handle_encode(C.byref(c), n, 0, C.byref(h)) == ob._abi.ERR_RANGE
    assert L.ouro_handle_encode(C.byref(c), 0, ppc, C.byref(h)) == ob._abi.ERR_RANGE
    a, b = C.c_uint32(), C.c_uint32()
    assert L.ouro_handle_decode(C.byref(c), n << 12, C.byref(a), C.byref(b)) == ob._abi.ERR_RANGE


def test_backoff_kats():
    O = oracle()
    for row in _load("spec_kats.json")["backoff"]:
        base, cap = row.get("base", 100), row.get("cap", 100000)
        assert ob.backoff_ns(row["policy"], row["attempt"], base, cap) == row["ns"]
        assert O.orc_backoff_ns(row["policy"], row["attempt"], base, cap) == row["ns"]
    for a in range(0, 70):
        assert ob.backoff_ns(1, a) == min(100 * 2 ** a, 100000)


def test_trial_means_kat():
    row = _load("spec_kats.json")["trial_means"][0]
    arr = (C.c_double * 10)(*row["ms"])
    a, s = C.c_double(), C.c_double()
    assert ob.lib().ouro_trial_means(arr, 10, C.byref(a), C.byref(s)) == 0
    assert a.value == pytest.approx(row["mean_all"], abs=0) or abs(a.value - 1.9) < 1e-12
    assert s.value == row["mean_subsequent"]
