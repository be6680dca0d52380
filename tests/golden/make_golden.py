"""Generate golden vectors by running the reference package itself.

Run in the build container (the reference is only mounted there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.json and tests/golden/golden.npz.  Nothing at test time reads
/root/reference; the tests only read these committed fixtures.  Every value below is an
output of the reference's own functions (batchrand.shuffle_batched, roll_batch, ...):
the oracle restatement (oracle/) and the CUDA product are both checked against them.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

import numpy as np

import batchrand as R
from batchrand.wordsource import splitmix64_stream

HERE = os.path.dirname(os.path.abspath(__file__))
MASK64 = (1 << 64) - 1


def array_seed(s: int, a: int) -> int:
    """SURVEY 8(c) per-array seed convention, via the reference's own splitmix64_stream."""
    return next(splitmix64_stream(((s << 32) | a) & MASK64))


class CountingSource(R.WordSource):
    def __init__(self, inner):
        self.inner = inner
        self.word_bits = inner.word_bits
        self.count = 0

    def next_word(self):
        self.count += 1
        return self.inner.next_word()


def sha_u32(seq) -> str:
    return hashlib.sha256(np.asarray(seq, dtype="<u4").tobytes()).hexdigest()


def sched_entries(s):
    return [[int(n), int(k)] for n, k in s.entries]


def main():
    t0 = time.time()
    out: dict = {}
    arrays: dict = {}

    # --- generators --------------------------------------------------------------
    seeds = [0, 1, 2, 5, 7, 42, 99, 1234, 12345, MASK64]
    out["pcg64"] = []
    for seed in seeds:
        src = R.make_source("pcg64", seed)
        st, inc = src.state, src.increment
        out["pcg64"].append({"seed": seed, "state": st, "inc": inc,
                             "words": [src.next_word() for _ in range(16)]})
    out["lehmer"] = []
    for seed in seeds:
        src = R.make_source("lehmer", seed)
        st = src.state
        out["lehmer"].append({"seed": seed, "state": st, "words": [src.next_word() for _ in range(8)]})
    out["splitmix64"] = [{"seed": s, "out": [v for _, v in zip(range(6), splitmix64_stream(s))]} for s in seeds]
    out["array_seed"] = [{"run_seed": s, "a": a, "seed": array_seed(s, a)}
                         for s in (1234, 99, 5, 7) for a in (0, 1, 2, 3, 255, 65535, (1 << 20) - 1)]
    # long stream checkpoint for jump-ahead: word 100000 of pcg64(5)
    src = R.make_source("pcg64", 5)
    for _ in range(100000):
        w = src.next_word()
    out["pcg64_seed5_word99999"] = w

    # --- bounded / batched --------------------------------------------------------
    rng = random.Random(20240809)
    out["falling_factorial"] = [[n, k, R.falling_factorial(n, k, 64)]
                                for n, k in ((6, 6), (7, 3), (5, 0), (2**32, 2), (1 << 19, 3), (1 << 14, 4),
                                             (1 << 11, 5), (1 << 9, 6), (4096, 4), (2048, 5), (64, 6), (4, 3))]
    out["threshold"] = [[b, R.threshold(R.BoundEncoding.of(b, 64))]
                        for b in (1, 2, 3, 6, 12, 52 * 51, 10**9 + 7, (1 << 64) - 1, 1 << 63, 65535 * 65534,
                                  R.falling_factorial(1 << 19, 3), R.falling_factorial(4096, 4))]
    dp = []
    for _ in range(200):
        k = rng.randrange(1, 7)
        bases = [rng.randrange(1, 1 << rng.choice((3, 8, 16, 20, 31))) for _ in range(k)]
        while np.prod([float(b) for b in bases]) >= 2.0**63:
            bases.pop()
        r0 = rng.getrandbits(64)
        digits, rk = R.digit_pass(r0, R.RadixBases.of(bases, 64))
        dp.append({"r0": r0, "bases": bases, "digits": list(digits), "rk": rk})
    out["digit_pass"] = dp

    # roll_batch on pcg64 streams, including rejection-heavy bases (products near 2^63/2^64)
    rb = []
    for seed, bases in ((11, (2, 6)), (12, (52, 51)), (13, (2**31 + 1, 2**31 - 1)), (14, (3, 5, 7, 11)),
                        (15, (65535, 65535, 65535, 65535)), (16, (2**32 - 1, 2**31 + 11)),
                        (17, (1 << 31, 1 << 31, 4)), (18, (1,)), (19, (2**32 - 1,)), (20, (6, 5, 4, 3, 2, 1))):
        src = R.make_source("pcg64", seed)
        spec = R.BatchSpec(R.RadixBases.of(bases, 64))
        res = []
        for _ in range(64):
            r = R.roll_batch(src, spec)
            res.append([list(r.digits), r.words_consumed, int(r.threshold_computed), r.final_remainder])
        rb.append({"seed": seed, "bases": list(bases), "results": res, "state_after": src.state})
    out["roll_batch"] = rb

    # --- C2 prefix: bounds from seed 7, rolls from hash(7, 1) ----------------------
    nb = 4096
    bsrc = R.make_source("pcg64", 7)
    bounds = [2 + R.roll_single(bsrc, (1 << 16) - 2) for _ in range(2 * nb)]
    rsrc = R.make_source("pcg64", array_seed(7, 1))
    rolls, wds = [], []
    for i in range(nb):
        r = R.roll_batch(rsrc, R.BatchSpec(R.RadixBases.of(bounds[2 * i:2 * i + 2], 64)))
        rolls.extend(r.digits)
        wds.append(r.words_consumed)
    arrays["c2_bounds"] = np.asarray(bounds, dtype=np.uint32)
    arrays["c2_rolls"] = np.asarray(rolls, dtype=np.uint32)
    arrays["c2_words"] = np.asarray(wds, dtype=np.uint8)
    out["c2"] = {"batches": nb, "roll_seed": array_seed(7, 1), "state_after": rsrc.state}

    # --- shuffles -------------------------------------------------------------------
    scheds = {
        "default": R.DEFAULT_SCHEDULE,
        "pair": R.PAIR_SCHEDULE,
        "max3": R.default_schedule(3),
        "max4": R.default_schedule(4),
        "max5": R.default_schedule(5),
        "head": R.ShuffleSchedule(((100, 2), (50, 3)), max_batch=3, word_bits=64),
        "wide": R.ShuffleSchedule(((1 << 12, 4), (200, 6), (40, 8)), max_batch=8, word_bits=64),
    }
    out["schedules"] = {k: {"entries": sched_entries(v), "max_batch": v.max_batch} for k, v in scheds.items()}
    sh = []
    ns = list(range(0, 71)) + [100, 127, 128, 129, 255, 256, 257, 300, 511, 512, 513, 1000, 2047, 2048, 2049,
                              4095, 4096, 4097, 10000, 16384, 16385, 65536]
    for n in ns:
        for name in ("default", "pair", "max3", "head", "wide"):
            if name != "default" and n > 4097:
                continue
            seed = rng.getrandbits(64)
            src = CountingSource(R.make_source("pcg64", seed))
            z = R.shuffle_batched(src, list(range(n)), scheds[name])
            rec = {"n": n, "schedule": name, "seed": seed, "words": src.count, "sha": sha_u32(z),
                   "head": z[:8], "tail": z[-8:]}
            if n <= 600:
                rec["perm"] = z
            sh.append(rec)
    out["shuffle_batched"] = sh
    un = []
    for n in list(range(0, 20)) + [64, 100, 1000, 4096]:
        seed = rng.getrandbits(64)
        src = CountingSource(R.make_source("pcg64", seed))
        z = R.shuffle_unbatched(src, list(range(n)))
        un.append({"n": n, "seed": seed, "words": src.count, "sha": sha_u32(z), "perm": z if n <= 600 else None})
    out["shuffle_unbatched"] = un

    # C1 (configs[0])
    c1 = {}
    src = CountingSource(R.make_source("pcg64", 42))
    z = R.shuffle_batched(src, list(range(10000)))
    c1["batched"] = {"words": src.count, "sha": sha_u32(z), "head": z[:8], "tail": z[-4:]}
    arrays["c1_batched"] = np.asarray(z, dtype=np.uint32)
    src = CountingSource(R.make_source("pcg64", 42))
    z = R.shuffle_unbatched(src, list(range(10000)))
    c1["unbatched"] = {"words": src.count, "sha": sha_u32(z), "head": z[:8]}
    arrays["c1_unbatched"] = np.asarray(z, dtype=np.uint32)
    out["c1"] = c1

    # C3 sample: arrays 0..255 of hash(1234, a), n=64 (full perms)
    c3 = np.empty((256, 64), dtype=np.uint8)
    c3w = []
    for a in range(256):
        src = CountingSource(R.make_source("pcg64", array_seed(1234, a)))
        c3[a] = R.shuffle_batched(src, list(range(64)))
        c3w.append(src.count)
    arrays["c3_perm_first256"] = c3
    out["c3_words_first256"] = c3w
    # a few high array indices
    c3hi = []
    for a in (1000, 65535, 524287, (1 << 20) - 1):
        src = CountingSource(R.make_source("pcg64", array_seed(1234, a)))
        z = R.shuffle_batched(src, list(range(64)))
        c3hi.append({"a": a, "perm": z, "words": src.count})
    out["c3_high"] = c3hi

    # C4 sample: n=4096, seeds hash(99, a)
    c4 = []
    for a in (0, 1, 2, 3, 100, 4095, 32768, 65535):
        src = CountingSource(R.make_source("pcg64", array_seed(99, a)))
        z = R.shuffle_batched(src, list(range(4096)))
        c4.append({"a": a, "sha": sha_u32(z), "words": src.count, "head": z[:8]})
    out["c4"] = c4

    # C5 sample: n=2^20 index permutations, seeds hash(5, a)
    c5 = []
    for a in (0, 255):
        src = CountingSource(R.make_source("pcg64", array_seed(5, a)))
        z = R.shuffle_batched(src, list(range(1 << 20)))
        c5.append({"a": a, "sha": sha_u32(z), "words": src.count, "head": z[:8]})
    out["c5"] = c5

    # partial_shuffle_batch cases (test_shuffle.py:85-144 style, 64-bit)
    pb = []
    for n, k in ((3, 3), (52, 2), (6, 2), (100, 6), (4096, 4)):
        for _ in range(4):
            seed = rng.getrandbits(64)
            src = R.make_source("pcg64", seed)
            z = list(range(n))
            u = R.falling_factorial(n, k, 64) + rng.choice((0, 0, 1000, 1 << 40))
            u = min(u, 1 << 64)
            u2 = R.partial_shuffle_batch(src, z, n, k, u)
            pb.append({"n": n, "k": k, "seed": seed, "u_in": u, "u_out": u2, "perm": z})
    out["partial_shuffle_batch"] = pb

    # Lehmer128 (wordsource.py:51-67) through the same hot path
    lsh = []
    for n in (2, 3, 5, 64, 100, 1000, 4096, 10000, 70000):
        for name in ("default", "pair"):
            seed = rng.getrandbits(64)
            src = CountingSource(R.make_source("lehmer", seed))
            z = R.shuffle_batched(src, list(range(n)), scheds[name])
            lsh.append({"n": n, "schedule": name, "seed": seed, "words": src.count, "sha": sha_u32(z)})
    src = CountingSource(R.LehmerSource(31337))
    R.shuffle_batched(src, list(range(1000)))
    out["lehmer_31337_n1000_words"] = src.count
    out["shuffle_batched_lehmer"] = lsh
    lun = []
    for n in (2, 17, 1000, 5000):
        seed = rng.getrandbits(64)
        src = CountingSource(R.make_source("lehmer", seed))
        z = R.shuffle_unbatched(src, list(range(n)))
        lun.append({"n": n, "seed": seed, "words": src.count, "sha": sha_u32(z)})
    out["shuffle_unbatched_lehmer"] = lun
    lrb = []
    for seed, bases in ((31, (6, 5)), (32, (2**32 - 1, 2**31 + 11)), (33, (1 << 16, 3, 5))):
        src = R.make_source("lehmer", seed)
        spec = R.BatchSpec(R.RadixBases.of(bases, 64))
        res = []
        for _ in range(48):
            r = R.roll_batch(src, spec)
            res.append([list(r.digits), r.words_consumed, int(r.threshold_computed), r.final_remainder])
        lrb.append({"seed": seed, "bases": list(bases), "results": res, "state_after": src.state})
    out["roll_batch_lehmer"] = lrb

    # ChaCha20 keystream (wordsource.py:102-164) through the same hot path
    out["chacha"] = []
    for seed in (0, 1, 3, 42, 12345, MASK64):
        src = R.make_source("chacha", seed)
        out["chacha"].append({"seed": seed, "key": list(src.key_words), "nonce": src.nonce,
                              "words": [src.next_word() for _ in range(20)]})
    rfc_key = tuple(int.from_bytes(bytes(range(32))[i:i + 4], "little") for i in range(0, 32, 4))
    out["chacha_block_rfc8439"] = {"key": list(rfc_key), "counter": (0x09000000 << 32) | 1, "nonce": 0x4A000000,
                                   "block": list(R.chacha_block(rfc_key, (0x09000000 << 32) | 1, 0x4A000000))}
    csh = []
    for n in (2, 3, 5, 64, 100, 1000, 4096, 10000, 70000):
        for name in ("default", "pair", "max3"):
            seed = rng.getrandbits(64)
            pre = rng.randrange(0, 9)  # start mid-block: words already drawn from the source
            src = R.make_source("chacha", seed)
            for _ in range(pre):
                src.next_word()
            cs = CountingSource(src)
            z = R.shuffle_batched(cs, list(range(n)), scheds[name])
            csh.append({"n": n, "schedule": name, "seed": seed, "pre": pre, "words": cs.count, "sha": sha_u32(z),
                        "counter_after": src.counter, "pos_after": src._pos})
    out["shuffle_batched_chacha"] = csh
    cun = []
    for n in (2, 17, 1000, 5000):
        seed = rng.getrandbits(64)
        src = CountingSource(R.make_source("chacha", seed))
        z = R.shuffle_unbatched(src, list(range(n)))
        cun.append({"n": n, "seed": seed, "words": src.count, "sha": sha_u32(z)})
    out["shuffle_unbatched_chacha"] = cun
    crb = []
    for seed, bases in ((41, (6, 5)), (42, (2**32 - 1, 2**31 + 11)), (43, (1 << 16, 3, 5)), (44, (7,))):
        src = R.make_source("chacha", seed)
        spec = R.BatchSpec(R.RadixBases.of(bases, 64))
        res = []
        for _ in range(48):
            r = R.roll_batch(src, spec)
            res.append([list(r.digits), r.words_consumed, int(r.threshold_computed), r.final_remainder])
        crb.append({"seed": seed, "bases": list(bases), "results": res, "counter_after": src.counter,
                    "pos_after": src._pos})
    out["roll_batch_chacha"] = crb

    # division-based baselines (shuffle.py:228-266, batched.py:126-128)
    nsh = []
    for gen in ("pcg64", "lehmer", "chacha"):
        for n in (0, 1, 2, 3, 4, 5, 64, 100, 101, 1000, 4096, 10000, 70001):
            seed = rng.getrandbits(64)
            src = CountingSource(R.make_source(gen, seed))
            z = R.shuffle_naive_batched(src, list(range(n)))
            rec = {"gen": gen, "n": n, "seed": seed, "words": src.count, "sha": sha_u32(z)}
            if n <= 100:
                rec["perm"] = z
            nsh.append(rec)
    out["shuffle_naive_batched"] = nsh
    nrb = []
    for seed, bases in ((51, (6, 5)), (52, (2**32 - 1, 2**31 + 11)), (53, (1 << 16, 3, 5)), (54, (10,)),
                        (55, (65535, 65521, 4099, 17))):
        src = CountingSource(R.make_source("pcg64", seed))
        rb = R.RadixBases.of(bases, 64)
        res = [list(R.roll_batch_naive(src, rb)) for _ in range(40)]
        nrb.append({"seed": seed, "bases": list(bases), "digits": res, "words": src.count})
    out["roll_batch_naive"] = nrb

    # cost model (cost_model.py): crossovers and schedules for a spread of
    # cost parameters, including GPU-like ones (expensive generator words / divisions)
    cm = []
    for rng_cost, div_cost, bits in ((2.0, 16.0, 64), (2.0, 16.0, 32), (1.0, 16.0, 64), (6.0, 20.0, 64),
                                     (3.0, 25.0, 64), (30.0, 20.0, 64), (60.0, 40.0, 64), (0.5, 4.0, 64),
                                     (10.0, 10.0, 32), (2.5, 70.0, 64)):
        params = R.CostParams(rng_cost=rng_cost, div_cost=div_cost, word_bits=bits)
        rec = {"rng_cost": rng_cost, "div_cost": div_cost, "bits": bits, "nk": {}}
        for k in range(2, 9 if bits == 64 else 5):
            try:
                rec["nk"][str(k)] = R.find_nk(k, params)
            except R.NoCrossover:
                rec["nk"][str(k)] = None
        try:
            rec["schedule6"] = [list(e) for e in R.build_schedule(params, 6 if bits == 64 else 4).entries]
        except (R.NoCrossover, ValueError) as e:
            rec["schedule6"] = type(e).__name__
        pts = ((1000, 2), (26573, 4), (815, 6), (146, 8), (70000, 3)) if bits == 64 else ((1000, 2), (500, 3), (100, 4))
        rec["costs"] = [[n, k, R.cost_per_roll(n, k, params)] for n, k in pts]
        cm.append(rec)
    out["cost_model"] = cm

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print(f"wrote golden fixtures in {time.time() - t0:.1f}s", file=sys.stderr)


if __name__ == "__main__":
    main()
