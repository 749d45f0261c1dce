"""Golden case table shared by make_golden.py (reference side) and the tests."""

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
