"""Shared test helpers: configs and seeded random op scripts (single lane and
whole warp) in the ouro_script_step format of include/ouro.h."""
import random

from paper_2504_18211_b200._abi import Config

VARIANTS = [(0, 0), (1, 0), (0, 1), (1, 1), (0, 2), (1, 2)]  # kAllVariants order (config.hpp:62-69)
NAMES = {(0, 0): "page", (1, 0): "chunk", (0, 1): "va-page", (1, 1): "va-chunk",
         (0, 2): "vl-page", (1, 2): "vl-chunk"}


def cfg(kind=0, flavor=0, heap=1 << 20, chunk=64 << 10, minp=16, maxp=8192, retries=8,
        backoff=0):
    return Config(heap, chunk, minp, maxp, flavor, kind, backoff, 0, retries, 100, 100000)


SIZES = [1, 4, 8, 15, 16, 17, 24, 32, 33, 64, 100, 128, 200, 256, 500, 512, 513, 1000, 1024,
         2000, 2048, 3000, 4096, 5000, 8000, 8192]


def random_script(seed, nsteps, warp=False, sizes=SIZES, p_free=0.45, bad=False, classes=None,
                  coalesced=False):
    """Returns list of (op, mask, args).  Frees reference earlier results by
    index (s*32+lane); `bad` injects double frees / invalid offsets."""
    rng = random.Random(seed)
    steps = []
    live = []
    size_pool = sizes if classes is None else [s for s in sizes if s in classes]
    for s in range(nsteps):
        args = [0] * 32
        if live and rng.random() < p_free:
            k = 1 if not warp else rng.randint(1, min(32, len(live)))
            lanes = rng.sample(range(32), k)
            mask = 0
            for ln in lanes:
                mask |= 1 << ln
                j = rng.randrange(len(live))
                live[j], live[-1] = live[-1], live[j]
                args[ln] = live.pop()
            if bad and rng.random() < 0.1:
                ln = lanes[0]
                r = rng.random()
                if r < 0.4 and s > 0:
                    args[ln] = rng.randrange(s * 32)          # maybe already freed -> DoubleFree
                elif r < 0.7:
                    args[ln] = (1 << 63) | (rng.randrange(1 << 20) | 1)  # misaligned offset
                else:
                    args[ln] = (1 << 63) | (1 << 40)         # out of heap
            steps.append((1, mask, args))
        else:
            if warp:
                k = rng.choice([1, 2, 5, 16, 31, 32])
                lanes = rng.sample(range(32), k)
                ncls = rng.choice([1, 1, 2, 3])
                menu = [rng.choice(size_pool) for _ in range(ncls)]
            else:
                lanes = [rng.randrange(32)]
                menu = [rng.choice(size_pool)]
            mask = 0
            for ln in lanes:
                mask |= 1 << ln
                args[ln] = rng.choice(menu)
                if bad and rng.random() < 0.02:
                    args[ln] = rng.choice([0, 8193, 1 << 40])
                live.append(s * 32 + ln)
            op = 2 if (coalesced and rng.random() < 0.3) else 0
            steps.append((op, mask, args))
    return steps


def single_lane_ops(steps):
    """Flatten a single-lane script into (op, value) pairs for the Python model."""
    out = []
    for op, mask, args in steps:
        ln = mask.bit_length() - 1
        out.append((op, ln, args[ln]))
    return out
