"""Golden case table shared by make_golden.py (reference side) and the tests.

Each case: (name, job factory, output config). Input files are cut from the
job's runs with the same block_size / restart_interval as the output.

* Scaled-down shapes of every BASELINE config plus edge cases (first block).
* BASELINE configs at their stated sizes where the oracle finishes in seconds:
  c1 (2 x 65,536, 16 B / 100 B), c2 (1 L1 + 10 L2 x 2 MB, 16 B / 1 KB),
  c4 literal (8 x 14,200, 24 B / 256 B).
* Planner stress: > 8,192 survivors and > 8,192 / > 16,384 output blocks
  (block_size 256), so both greedy chains compose over several tiles and
  groups; one case puts > 90 K entries in ONE SST (filter and index blocks
  far above 48 KiB).
* Oversized values (4-12 KiB: single-entry blocks above block_size), and
  bits_per_key 1 / 7 / 13.
* 200 SPEC-A1 random jobs and 24 small mixed jobs.
"""

from oracle import jobgen

SMALL_OUT = dict(sst_size_target=48 * 1024)

CASES = [
    ("c1_small", lambda: jobgen.c1(n=3000), dict(sst_size_target=96 * 1024)),
    ("c1_dup_tomb", lambda: jobgen.c1(n=3000, seed=0xC11, dup_frac=0.5, del_frac=0.2),
     dict(sst_size_target=96 * 1024)),
    ("c2_small", lambda: jobgen.c2(n_upper=1964, upper_target=200 * 1024), dict(sst_size_target=512 * 1024)),
    ("c3_small", lambda: jobgen.c3(n=6000, sst_target=96 * 1024), dict(sst_size_target=128 * 1024)),
    ("c3_deeper", lambda: jobgen.c3(n=3000, seed=0xC33, sst_target=64 * 1024,
                                    deeper=[(b"\x20" * 16, b"\x9f" * 16)]), SMALL_OUT),
    ("c4_small", lambda: jobgen.c4(n_per_file=400, files=8), dict(sst_size_target=256 * 1024)),
    ("c4_onefile", lambda: jobgen.c4(n_per_file=700, files=1, seed=0xC44), SMALL_OUT),
    ("ri4_bs1024", lambda: jobgen.c3(n=2500, seed=0xAB, sst_target=40 * 1024),
     dict(sst_size_target=20 * 1024, block_size=1024, restart_interval=4)),
    ("all_tombstones", lambda: jobgen.c1(n=500, seed=0xDD, dup_frac=1.0, del_frac=1.0), SMALL_OUT),
] + [
    (f"mixed{s}", (lambda s=s: jobgen.mixed(s)), dict(sst_size_target=8 * 1024 + 512 * (s % 7)))
    for s in range(24)
]

# BASELINE configs at their stated sizes (BASELINE.json configs[0], [1], [3])
FULL_CASES = [
    ("c1_full", lambda: jobgen.c1(), {}),
    ("c2_full", lambda: jobgen.c2(), {}),
    ("c4_literal", lambda: jobgen.c4(), {}),
]

EDGE_CASES = [
    # > 8,192 survivors and ~17 K output blocks of 256 B, cut into 32 KiB SSTs:
    # the block chain spans 15 tiles in 4 groups, the SST chain 3 tiles in 2 groups.
    ("multitile_ssts", lambda: jobgen.c3(n=150000, seed=0xA1, vlen=8, sst_target=2**31),
     dict(block_size=256, sst_size_target=32 * 1024)),
    # ~92 K entries in ONE output SST: 115 KB filter, ~420 KB index.
    ("multitile_one_sst", lambda: jobgen.c3(n=115000, seed=0xA2, vlen=8, sst_target=2**31),
     dict(block_size=256, sst_size_target=2**31)),
    ("values_4k_12k", lambda: jobgen.values_job(), dict(sst_size_target=1 << 20)),
    ("values_4k_12k_small_sst", lambda: jobgen.values_job(n=300, seed=0xB17, del_frac=0.3),
     dict(sst_size_target=64 * 1024, restart_interval=3)),
    ("bpk1", lambda: jobgen.c3(n=3000, seed=0xB1, sst_target=64 * 1024), dict(sst_size_target=96 * 1024,
                                                                               bits_per_key=1)),
    ("bpk7", lambda: jobgen.c3(n=3000, seed=0xB7, sst_target=64 * 1024), dict(sst_size_target=96 * 1024,
                                                                               bits_per_key=7)),
    ("bpk13", lambda: jobgen.c3(n=3000, seed=0xB13, sst_target=64 * 1024), dict(sst_size_target=96 * 1024,
                                                                                 bits_per_key=13)),
    ("bpk13_one_sst", lambda: jobgen.c3(n=20000, seed=0xB14, vlen=16, sst_target=2**31),
     dict(sst_size_target=2**31, bits_per_key=13)),
]

SPEC_A1_CASES = [
    (f"spec_a1_{s}", (lambda s=s: jobgen.spec_a1(s)), dict(sst_size_target=[16, 64, 256, 1024][s % 4] * 1024))
    for s in range(200)
]

ALL_CASES = CASES + FULL_CASES + EDGE_CASES + SPEC_A1_CASES

# Generic user-key lengths (keys.py:60-63: a shorter prefix sorts first;
# blocks.py:33-58: shared prefixes may run into the trailer).
VARKEY_CASES = [
    (f"varkey{s}", (lambda s=s: jobgen.varkey(s)), dict(sst_size_target=[8, 32, 2**21][s % 3] * 1024))
    for s in range(12)
] + [
    (f"varkey_short{s}", (lambda s=s: jobgen.varkey(100 + s, max_len=6, n_space=300)),
     dict(sst_size_target=8 * 1024, restart_interval=[16, 3, 1][s % 3]))
    for s in range(6)
] + [
    ("fixed40", lambda: jobgen.c4(n_per_file=1500, files=3, seed=0x40, klen=40, vlen=100),
     dict(sst_size_target=64 * 1024)),
    ("fixed64", lambda: jobgen.c3(n=2000, seed=0x64, klen=64, sst_target=64 * 1024), dict(sst_size_target=96 * 1024)),
    ("fixed1", lambda: jobgen.c4(n_per_file=200, files=4, seed=0x41, klen=1, vlen=50), {}),
    ("fixed9_ri2", lambda: jobgen.c3(n=2000, seed=0x09, klen=9, sst_target=32 * 1024),
     dict(sst_size_target=40 * 1024, restart_interval=2)),
] + [
    # user keys past the 71-byte var record: the long records (kVarWLong, <= 255 bytes)
    (f"varkey_long{s}", (lambda s=s: jobgen.varkey(200 + s, max_len=[120, 200, 255][s % 3], n_space=300)),
     dict(sst_size_target=[16, 64][s % 2] * 1024, restart_interval=[16, 4][s % 2]))
    for s in range(6)
] + [
    ("fixed100", lambda: jobgen.c3(n=1500, seed=0x100, klen=100, sst_target=48 * 1024), dict(sst_size_target=64 * 1024)),
]

ALL_CASES = ALL_CASES + VARKEY_CASES
