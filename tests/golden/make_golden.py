"""Generate the committed golden fixtures (run here, where /root/reference exists).

config_validate.json : HeapConfig::validate outcome + message, num_chunks and
                       max_pages_per_chunk for a grid of configs, produced by the
                       REFERENCE's own proj/src/config.cpp (oracle/_ref).
variants.json        : kAllVariants order and variant_name / variant_from_name
                       from the same reference build.
spec_kats.json       : the SPEC's literal known-answer examples
                       (/root/reference/SPEC.md line cited per entry).

Usage: python tests/golden/make_golden.py
"""
import ctypes as C
import itertools
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_lib import ref  # noqa: E402
from paper_2504_18211_b200._abi import Config  # noqa: E402


def config_grid():
    vals = [0, 1, 3, 8, 16, 24, 1000, 1024, 3 << 10, 8192, 64 << 10, 1 << 20, 64 << 20, 1 << 30,
            1 << 34, 1 << 40, 1 << 44, 1 << 50]
    rng = random.Random(2504_18211)
    out = []
    # structured sweep around the defaults
    for heap, chunk, minp, maxp in itertools.product(
            [64 << 10, 1 << 20, 64 << 20, 1 << 30, 16 << 30, 1 << 40, 3 << 20],
            [16, 8192, 64 << 10, 3 << 10, 1 << 20, 1 << 30],
            [1, 16, 24, 64], [16, 8192, 1 << 20, 1000]):
        for retries in (0, 1, 64):
            out.append((heap, chunk, minp, maxp, retries))
    for _ in range(1000):
        out.append((rng.choice(vals), rng.choice(vals), rng.choice(vals), rng.choice(vals),
                    rng.choice([0, 1, 64, 2 ** 32 - 1])))
    return out


def main():
    R = ref()
    if R is None:
        sys.exit("reference build (oracle/_ref) unavailable")
    rows = []
    msgs = [""]
    msg = C.create_string_buffer(256)
    for heap, chunk, minp, maxp, retries in config_grid():
        c = Config(heap, chunk, minp, maxp, 0, 0, 0, 0, retries, 100, 100000)
        rc = R.ref_validate(C.byref(c), msg, 256)
        m = msg.value.decode() if rc else ""
        if m not in msgs:
            msgs.append(m)
        rows.append([heap, chunk, minp, maxp, retries, int(rc == 0), msgs.index(m),
                     R.ref_num_chunks(C.byref(c)) if chunk else -1,
                     R.ref_max_pages_per_chunk(C.byref(c)) if minp else -1])
    with open(os.path.join(HERE, "config_validate.json"), "w") as f:
        json.dump({"source": "/root/reference/proj/src/config.cpp via oracle/_ref",
                   "columns": ["heap", "chunk", "min", "max", "retries", "valid", "msg",
                               "num_chunks", "max_pages_per_chunk"],
                   "messages": msgs, "rows": rows}, f, separators=(",", ":"))
    kinds = (C.c_uint8 * 8)()
    flavs = (C.c_uint8 * 8)()
    n = R.ref_all_variants(kinds, flavs)
    names = []
    buf = C.create_string_buffer(32)
    for i in range(n):
        R.ref_variant_name(kinds[i], flavs[i], buf, 32)
        names.append({"kind": kinds[i], "flavor": flavs[i], "name": buf.value.decode()})
    lay = (C.c_uint64 * 9)()
    R.ref_layout(lay)
    dflt = Config()
    R.ref_default(C.byref(dflt))
    with open(os.path.join(HERE, "variants.json"), "w") as f:
        json.dump({"all_variants": names, "layout": list(lay),
                   "defaults": [dflt.heap_bytes, dflt.chunk_bytes, dflt.min_page_bytes,
                                dflt.max_page_bytes, dflt.queue_flavor, dflt.allocator_kind,
                                dflt.backoff, dflt.max_retries, dflt.sleep_base_ns,
                                dflt.sleep_cap_ns]}, f, indent=1)
    print(f"wrote {len(rows)} validate rows, {n} variants")


if __name__ == "__main__":
    main()
