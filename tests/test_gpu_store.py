"""Store integration with the reference's own LSM objects:
``pick_compaction`` (version.py:175) → GPU ``run_compaction`` (outputs named by
the reference's ``VersionSet.new_file_id``) → ``apply_compaction_result``
(version.py:377, MANIFEST edit), plus the pipelined ``run_compactions`` over
several golden jobs and the zero-copy ``StagedInput`` path.

The reference package comes from ``baseline/_ref`` (pip-installed from
/root/reference; it travels with the repo snapshot) — skipped without it."""

import os
import random

import pytest

import bench_ref
from oracle import jobgen
from oracle import luda_oracle as O

pytestmark = pytest.mark.gpu

R = bench_ref.load_reference()


@pytest.fixture(scope="module")
def dev():
    from paper_2004_03054_b200 import DeviceConfig, make_device
    d = make_device(DeviceConfig(backend="b200"))
    yield d
    d.close()


def _sst(R, pairs, vset, level):
    fid = vset.new_file_id()
    data, meta = R.sst.build_sst(pairs, file_id=fid, level=level)
    with open(os.path.join(vset.directory, f"{fid}.sst"), "wb") as f:
        f.write(data)
    return meta


@pytest.mark.skipif(R is None, reason="reference not installed in baseline/_ref")
def test_pick_run_apply_with_reference_versionset(dev, tmp_path):
    import luda.version as RV
    from paper_2004_03054_b200 import run_compaction
    from paper_2004_03054_b200.config import StoreConfig
    rng = random.Random(0x5707E)
    vset = RV.VersionSet(str(tmp_path))
    space = sorted({rng.randbytes(16) for _ in range(3000)})
    seq = 1
    added = []
    # one L2 file over the middle of the key space: tombstones there must survive (D12)
    mid = space[1000:1600:3]
    added.append(_sst(R, [(R.keys.encode_key(k, seq + i, 1), b"deep") for i, k in enumerate(mid)], vset, 2))
    seq += len(mid)
    # two L1 files, then five overlapping L0 files (newest = highest file id)
    l1 = sorted(rng.sample(space, 1200))
    for part in (l1[:600], l1[600:]):
        added.append(_sst(R, [(R.keys.encode_key(k, seq + i, 1), rng.randbytes(100)) for i, k in enumerate(part)],
                          vset, 1))
        seq += len(part)
    for _ in range(5):
        ks = sorted(rng.sample(space, 500))
        pairs = []
        for k in ks:
            dele = rng.random() < 0.15
            pairs.append((R.keys.encode_key(k, seq, 0 if dele else 1), b"" if dele else rng.randbytes(80)))
            seq += 1
        added.append(_sst(R, pairs, vset, 0))
    vset.log_and_apply(RV.VersionEdit(added=added, last_seq=seq))
    cfg = R.config.StoreConfig(l0_compaction_trigger=4, background=False, sst_size_target=64 * 1024)
    job = RV.pick_compaction(vset.current, cfg)
    assert job is not None and job.source_level == 0 and len(job.lower) == 5 and len(job.upper) == 2
    outs, stats = run_compaction(job, dev, directory=str(tmp_path), new_file_id=vset,
                                 config=StoreConfig(sst_size_target=64 * 1024))
    # byte parity with the reference's own composition over the same files (deeper = covers_below spans)
    files = [open(os.path.join(tmp_path, f"{m.file_id}.sst"), "rb").read() for m in job.lower + job.upper]
    deeper = [(R.keys.user_key_of(f.smallest), R.keys.user_key_of(f.largest))
              for lv in job.version.levels[job.target_level + 1:] for f in lv]
    want = bench_ref.ref_compact(R, files, deeper=deeper, sst_size_target=64 * 1024)
    assert [d for d, _ in outs] == want
    metas = []
    for data, m in outs:
        with open(os.path.join(tmp_path, f"{m.file_id}.sst"), "wb") as f:
            f.write(data)
        metas.append(R.sst.SstMeta(file_id=m.file_id, file_size=m.file_size, smallest=m.smallest,
                                   largest=m.largest, level=m.level))
    ids = [m.file_id for m in metas]
    assert len(set(ids)) == len(ids) and min(ids) > max(m.file_id for m in added)  # VersionSet-allocated
    v2 = RV.apply_compaction_result(vset, job, metas)
    assert not v2.levels[0] and [m.file_id for m in v2.levels[1]] == ids
    # MANIFEST replay reproduces the new version; the reference's Table reads every output
    vset.close()
    again = RV.VersionSet(str(tmp_path))
    assert [[m.file_id for m in lv] for lv in again.current.levels] == [[m.file_id for m in lv] for lv in v2.levels]
    got = []
    for m in again.current.levels[1]:
        t = R.sst.open_sst(os.path.join(tmp_path, f"{m.file_id}.sst"), file_id=m.file_id)
        got += list(t.scan())
    assert len(got) == stats.n_out
    again.close()
    # SPEC.md:360 job-stats row
    row = stats.csv_row().split(",")
    assert len(row) == len(stats.CSV_COLUMNS) and int(row[3]) == sum(len(f) for f in files)


def test_run_compactions_pipeline_matches_oracle(dev):
    """Several different jobs through the double-buffered pipeline (jobs k+1
    staged while k compacts and k-1 streams out), from bytes inputs and from a
    pinned StagedInput; outputs are memoryviews valid until the next step."""
    from paper_2004_03054_b200 import run_compactions
    from paper_2004_03054_b200.compaction import StagedInput
    from paper_2004_03054_b200.config import StoreConfig
    from paper_2004_03054_b200.version import CompactionJob, SstMeta, Version
    from tests.golden.cases import ALL_CASES
    cases = {n: (mk, cfg) for n, mk, cfg in ALL_CASES}
    names = ["c3_small", "c4_small", "mixed3", "c1_dup_tomb", "varkey2", "c2_small"]
    jobs, wants, stage_keep = [], [], []
    fid = 1
    for i, name in enumerate(names):
        mk, cfg = cases[name]
        spec = mk()
        lower, upper = jobgen.materialize(spec)
        wants.append(O.reference_compact(lower + upper, deeper=spec.deeper, sst_size_target=256 * 1024))
        metas = []
        for f in lower + upper:
            metas.append(SstMeta(file_id=fid, file_size=len(f), smallest=b"", largest=b"",
                                 level=spec.source_level if len(metas) < len(lower) else spec.target_level))
            fid += 1
        ver = Version()
        for lo, hi in spec.deeper:
            ver.levels[spec.target_level + 1].append(SstMeta(0, 0, lo + bytes(8), hi + bytes(8), spec.target_level + 1))
        job = CompactionJob(source_level=spec.source_level, lower=metas[:len(lower)], upper=metas[len(lower):],
                            target_level=spec.target_level, version=ver)
        if i % 2:
            st = StagedInput([len(f) for f in lower + upper])
            for v, f in zip(st.views, lower + upper):
                v[:] = f
            stage_keep.append(st)
            jobs.append((job, st))
        else:
            jobs.append((job, {m.file_id: bytearray(f) for m, f in zip(metas, lower + upper)}))
    seen = 0
    inputs = {}
    for _, inp in jobs:
        if isinstance(inp, dict):
            inputs.update(inp)
    seq = [j if isinstance(inp, StagedInput) else j for j, inp in jobs]
    it = run_compactions([(j, inp) if isinstance(inp, StagedInput) else j for j, inp in jobs], dev,
                         inputs=inputs, config=StoreConfig(sst_size_target=256 * 1024))
    all_ids = []
    for (outs, stats), want in zip(it, wants):
        assert [bytes(d) for d, _ in outs] == [w[0] for w in want]
        assert [(m.smallest, m.largest) for _, m in outs] == [(w[1], w[2]) for w in want]
        all_ids += [m.file_id for _, m in outs]
        seen += 1
    assert seen == len(names) and len(set(all_ids)) == len(all_ids)
    for st in stage_keep:
        st.free()
