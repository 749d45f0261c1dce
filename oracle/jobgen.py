"""Seeded synthetic compaction jobs (the shapes of BASELINE.json configs) —
TEST INFRASTRUCTURE ONLY (tests/, bench.py cpu legs, golden generation).

A job is described as sorted *runs* of (internal_key, value) pairs plus the
level wiring; :func:`materialize` cuts each run into SST files with a table
builder (the oracle's here, the reference's in ``tests/golden/make_golden.py``)
using the SizeOverflowError cut rule. Keys are uniform random bytes from
``random.Random(seed)`` as SURVEY.md §8(d) prescribes; newer runs carry
strictly higher, globally unique sequence numbers.
"""

from __future__ import annotations

import random
from dataclasses import dataclass, field

from oracle import luda_oracle as O


@dataclass
class RunSpec:
    pairs: list            # sorted (ikey, value)
    level: int             # level the run's files live on
    sst_target: int        # cut size used to split the run into files


@dataclass
class JobSpec:
    name: str
    lower: list            # RunSpecs at source level (L0: one run per file)
    upper: list            # RunSpecs at target level
    source_level: int
    target_level: int
    deeper: list = field(default_factory=list)   # [(lo_user, hi_user)] below target

    def runs(self):
        return self.lower + self.upper


def _distinct_keys(rng, n, klen):
    seen = set()
    while len(seen) < n:
        seen.add(rng.randbytes(klen))
    return sorted(seen)


def _run(keys_seq_kind, rng, vlen, vlen_jitter=0):
    pairs = []
    for uk, seq, kind in keys_seq_kind:
        if kind == O.KIND_DELETE:
            v = b""
        else:
            n = vlen if not vlen_jitter else max(0, vlen + rng.randint(-vlen_jitter, vlen_jitter))
            v = rng.randbytes(n)
        pairs.append((O.make_ikey(uk, seq, kind), v))
    pairs.sort(key=lambda kv: O.order_key(kv[0]))
    return pairs


def c1(n=65536, seed=0xC1, klen=16, vlen=100, dup_frac=0.0, del_frac=0.0):
    """2 L0 SSTs x n distinct keys (config[0]); optional overwrite/tombstone mix."""
    rng = random.Random(seed)
    keys_old = _distinct_keys(rng, n, klen)
    n_dup = int(n * dup_frac)
    dups = rng.sample(keys_old, n_dup) if n_dup else []
    fresh = set(keys_old)
    new_keys = list(dups)
    while len(new_keys) < n:
        k = rng.randbytes(klen)
        if k not in fresh:
            fresh.add(k)
            new_keys.append(k)
    old = [(k, 1 + i, O.KIND_PUT) for i, k in enumerate(keys_old)]
    new = []
    for i, k in enumerate(sorted(new_keys)):
        kind = O.KIND_DELETE if rng.random() < del_frac else O.KIND_PUT
        new.append((k, n + 1 + i, kind))
    big = 2**31
    return JobSpec("c1", lower=[RunSpec(_run(new, rng, vlen), 0, big),
                                RunSpec(_run(old, rng, vlen), 0, big)],
                   upper=[], source_level=0, target_level=1)


def c2(n_upper=19640, seed=0xC2, klen=16, vlen=1024, upper_target=2 * 2**20, lower_frac=0.1):
    """1 L1 SST vs 10 overlapping L2 SSTs of ~2 MB (config[1])."""
    rng = random.Random(seed)
    ukeys = _distinct_keys(rng, n_upper, klen)
    n_lower = max(1, int(n_upper * lower_frac))
    lo_keys = set()
    while len(lo_keys) < n_lower:
        lo_keys.add(rng.randbytes(klen))
    upper = [(k, 1 + i, O.KIND_PUT) for i, k in enumerate(ukeys)]
    lower = [(k, n_upper + 1 + i, O.KIND_PUT) for i, k in enumerate(sorted(lo_keys))]
    return JobSpec("c2", lower=[RunSpec(_run(lower, rng, vlen), 1, 2**31)],
                   upper=[RunSpec(_run(upper, rng, vlen), 2, upper_target)],
                   source_level=1, target_level=2)


def c3(n=2**25, seed=0xC3, klen=16, vlen=128, del_frac=0.2, sst_target=4 * 2**20,
       deeper=None):
    """Overwrite-heavy: Li run overwrites every key of the Li+1 run, 20% deletes (config[2])."""
    rng = random.Random(seed)
    keys = _distinct_keys(rng, n, klen)
    upper = [(k, 1 + i, O.KIND_PUT) for i, k in enumerate(keys)]
    lower = []
    for i, k in enumerate(keys):
        kind = O.KIND_DELETE if rng.random() < del_frac else O.KIND_PUT
        lower.append((k, n + 1 + i, kind))
    return JobSpec("c3", lower=[RunSpec(_run(lower, rng, vlen), 1, sst_target)],
                   upper=[RunSpec(_run(upper, rng, vlen), 2, sst_target)],
                   source_level=1, target_level=2, deeper=deeper or [])


def c4(n_per_file=14200, files=8, seed=0xC4, klen=24, vlen=256, sst_target=2**31):
    """8 overlapping L0 files of random keys (config[3]); file i newer than i+1."""
    rng = random.Random(seed)
    runs = []
    seq = files * n_per_file
    for f in range(files):
        ks = _distinct_keys(rng, n_per_file, klen)
        trip = []
        for k in ks:
            trip.append((k, seq, O.KIND_PUT))
            seq -= 1
        runs.append(RunSpec(_run(trip, rng, vlen), 0, sst_target))
    return JobSpec("c4", lower=runs, upper=[], source_level=0, target_level=1)


def mixed(seed, n_files=None, max_keys=400, key_space=600, klen=16, vlen_max=300,
          del_frac=0.1, level0=True):
    """SPEC A1-style random job: 1-6 L0 files over a shared key space,
    variable value sizes (0..vlen_max), 0-20% tombstones, some overwrites."""
    rng = random.Random(seed)
    n_files = n_files or rng.randint(1, 6)
    space = _distinct_keys(rng, key_space, klen)
    seq = 1
    runs = []
    for _ in range(n_files):
        cnt = rng.randint(1, max_keys)
        ks = sorted(rng.sample(space, min(cnt, len(space))))
        trip = []
        for k in ks:
            kind = O.KIND_DELETE if rng.random() < del_frac else O.KIND_PUT
            trip.append((k, seq, kind))
            seq += 1
        pairs = []
        for uk, s, kind in trip:
            v = b"" if kind == O.KIND_DELETE else rng.randbytes(rng.randint(0, vlen_max))
            pairs.append((O.make_ikey(uk, s, kind), v))
        pairs.sort(key=lambda kv: O.order_key(kv[0]))
        runs.append(RunSpec(pairs, 0, 2**31))
    runs.reverse()  # newest file first, like L0 in a Version
    return JobSpec(f"mixed{seed}", lower=runs, upper=[], source_level=0, target_level=1)


def materialize(job: JobSpec, builder=O.build_tables_split, **cfg):
    """Cut every run into files; returns (lower_files, upper_files) as bytes lists."""
    def files_of(run):
        return [f for f, _, _ in builder(run.pairs, sst_size_target=run.sst_target, **cfg)]
    lower = [f for r in job.lower for f in files_of(r)]
    upper = [f for r in job.upper for f in files_of(r)]
    return lower, upper


def values_job(n=400, seed=0xB16, klen=16, vmin=4096, vmax=12288, del_frac=0.1, sst_target=2**31):
    """Two overlapping runs (Li newer than Li+1) with value lengths uniform in
    [vmin, vmax]: values of 4-12 KiB make single-entry blocks larger than the
    4 KiB block size (sst.py:153-177 lets one entry overflow a block)."""
    rng = random.Random(seed)
    keys = _distinct_keys(rng, n, klen)
    upper = [(k, 1 + i, O.KIND_PUT) for i, k in enumerate(keys)]
    sub = sorted(rng.sample(keys, n // 2))
    lower = [(k, n + 1 + i, O.KIND_DELETE if rng.random() < del_frac else O.KIND_PUT) for i, k in enumerate(sub)]

    def run(trip):
        pairs = []
        for uk, seq, kind in trip:
            v = b"" if kind == O.KIND_DELETE else rng.randbytes(rng.randint(vmin, vmax))
            pairs.append((O.make_ikey(uk, seq, kind), v))
        return pairs
    return JobSpec("values", lower=[RunSpec(run(lower), 1, sst_target)],
                   upper=[RunSpec(run(upper), 2, sst_target)], source_level=1, target_level=2)


def spec_a1(seed):
    """SPEC A1 random job: 1-6 L0 SSTs over a shared key space,
    value sizes 64 B - 4 KiB, 0-20% tombstones, overwrites across files."""
    rng = random.Random(0xA1000 + seed)
    n_files = rng.randint(1, 6)
    del_frac = rng.uniform(0.0, 0.2)
    space = _distinct_keys(rng, rng.randint(50, 400), 16)
    seq = 1
    runs = []
    for _ in range(n_files):
        ks = sorted(rng.sample(space, rng.randint(1, min(200, len(space)))))
        pairs = []
        for k in ks:
            kind = O.KIND_DELETE if rng.random() < del_frac else O.KIND_PUT
            v = b"" if kind == O.KIND_DELETE else rng.randbytes(rng.randint(64, 4096))
            pairs.append((O.make_ikey(k, seq, kind), v))
            seq += 1
        runs.append(RunSpec(pairs, 0, 2**31))
    runs.reverse()  # newest file first, like L0 in a Version
    return JobSpec(f"spec_a1_{seed}", lower=runs, upper=[], source_level=0, target_level=1)


def _varkeys(rng, n, max_len):
    """Distinct user keys of mixed lengths 0..max_len, rich in prefix pairs
    (k and k + suffix) and in bytes that collide with trailer bytes, so shared
    prefixes run into the 8-byte trailer (blocks.py:33-58, keys.py:60-63)."""
    out = set()
    alphabet = bytes([0, 1, 2, 0x7F, 0x80, 0xFE, 0xFF]) + b"abc"
    while len(out) < n:
        r = rng.random()
        if out and r < 0.35:
            base = rng.choice(sorted(out))
            if rng.random() < 0.5 and len(base) < max_len:   # extend: base is a prefix of the new key
                k = base + bytes(rng.choice(alphabet) for _ in range(rng.randint(1, min(8, max_len - len(base)))))
            else:                                             # truncate: new key is a prefix of base
                k = base[:rng.randint(0, len(base))]
        elif r < 0.6:
            k = bytes(rng.choice(alphabet) for _ in range(rng.randint(0, max_len)))
        else:
            k = rng.randbytes(rng.randint(0, max_len))
        out.add(k)
    return sorted(out)


def varkey(seed, max_len=64, n_space=500, n_files=None):
    """Mixed user-key lengths 0..max_len in one job (L0 files over one key space)."""
    rng = random.Random(0x7A4000 + seed)
    space = _varkeys(rng, n_space, max_len)
    n_files = n_files or rng.randint(2, 5)
    seq = 1
    runs = []
    for _ in range(n_files):
        ks = sorted(rng.sample(space, rng.randint(1, len(space))))
        trip = []
        for k in ks:
            trip.append((k, seq, O.KIND_DELETE if rng.random() < 0.1 else O.KIND_PUT))
            seq += 1
        runs.append(RunSpec(_run(trip, rng, 40, vlen_jitter=40), 0, 2**31))
    runs.reverse()
    return JobSpec(f"varkey{seed}", lower=runs, upper=[], source_level=0, target_level=1)
