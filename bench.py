"""LUDA compaction benchmark on B200 (BASELINE.json metric: compaction input
MB/s and keys/s per B200; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl b200|reference]

A step = one full compaction job (luda_compact: parse → decode → merge/resolve
→ plan → encode → filter/index/footer) over the config's input SSTs.
* value : device-resident (inputs already in HBM, outputs left in HBM).
* e2e   : through the same C ABI with HOST buffers — pinned H2D of every input
          file on the in_lower/in_upper streams, the job, D2H of every output.
Inputs are synthesised on the GPU with this package's own SST builder (the
bytes equal SstBuilder's; tests/test_gpu_parity.py) — 9.7 GB for c3, far
larger than L2, so no L2 flush is needed between steps.
Multi-GPU (torchrun): one process per GPU, each compacting its own key range
(weak scaling); timing is the max over ranks.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    # name: (description, generator kwargs)
    "c3": "Overwrite-heavy compaction: 64M KV pairs, 50% duplicate keys across runs plus 10% tombstones, "
          "16B/128B, 1 B200",
    "c1": "L0->L1 compaction of 2 input SSTs x 64K KV pairs (16B keys, 100B values, 4KB blocks)",
}

METRIC = "compaction input MB/s"


def workload_text(keys, world):
    """The c3 description with the actual job size (--keys other than 2^25 is a smaller c3-shaped job)."""
    t = CONFIGS["c3"]
    if keys != 1 << 25:
        t = t.replace("64M KV pairs", f"{2 * keys / 2**20:g}M KV pairs (c3-shaped, reduced from 64M)")
    if world > 1:
        t = t.replace(", 1 B200", "") + (f" per GPU; global job = {world} key-range shards "
                                         "(5th BASELINE config's subcompaction scheme)")
    return t
MIB4 = 4 * 2**20


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


# --------------------------------------------------------------------------------------------
# clocks
# --------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------------------------
# GPU workload synthesis (c3): two sorted runs of SSTs built on the device
# --------------------------------------------------------------------------------------------
class Workload:
    pass


def synth_c3(n_keys, seed, device_index, del_frac=0.2, vlen=128, klen=16, sst_target=MIB4, shard=0, nshards=1,
             keep_truth=False):
    import torch

    from paper_2004_03054_b200 import _native
    from paper_2004_03054_b200.flush import result_files  # noqa: F401 (keeps import graph honest)
    L = _native.lib(device_index)
    dev = torch.device("cuda", device_index)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    n = n_keys
    # sorted distinct 16-byte keys: sorted random 64-bit prefix (sign-flipped → unsigned order) + random suffix.
    # With nshards > 1 (multi-GPU weak scaling) the prefix's top log2(nshards) bits are the shard index, so the
    # ranks hold disjoint key ranges of one global job.
    b = nshards.bit_length() - 1
    assert 1 << b == nshards
    while True:
        hi = torch.randint(-2**63, 2**63 - 1, (n,), generator=g, device=dev, dtype=torch.int64)
        if b:
            hi = (hi >> b) & ((1 << (64 - b)) - 1)   # logical shift: [0, 2^(64-b)), sorts as signed == unsigned
        hi, _ = torch.sort(hi)
        if bool((hi[1:] != hi[:-1]).all()):
            break
    if b:
        prefix = shard << (64 - b)
        hi = hi | (prefix - 2**64 if prefix >= 2**63 else prefix)
    else:
        hi = hi ^ torch.tensor(-2**63, dtype=torch.int64, device=dev)
    lo = torch.randint(-2**63, 2**63 - 1, (n,), generator=g, device=dev, dtype=torch.int64)
    words = torch.stack([hi, lo], 1).contiguous()
    keys = words.view(torch.uint8).view(n, 2, 8).flip(2).reshape(n * 16).contiguous()
    assert klen == 16
    vbytes = n * vlen + 4096
    values = torch.empty(vbytes, dtype=torch.uint8, device=dev).random_(0, 256, generator=g)
    idx = torch.arange(n, device=dev, dtype=torch.int64)
    # Li+1 (upper): every key, seq 1..n, Put
    tr_up = ((idx + 1) << 8) | 1
    voff_up = idx * vlen + 64
    vlen_up = torch.full((n,), vlen, dtype=torch.int32, device=dev)
    # Li (lower): same keys, seq n+1.., del_frac Deletes with empty values
    is_del = torch.rand(n, generator=g, device=dev) < del_frac
    tr_lo = ((idx + n + 1) << 8) | (~is_del).to(torch.int64)
    voff_lo = idx * vlen + 64 + 61
    vlen_lo = torch.where(is_del, 0, vlen).to(torch.int32)
    torch.cuda.synchronize(dev)
    s = ctypes.c_void_p()
    _native.check(L.luda_stream_create(ctypes.byref(s)))

    def build(tr, voff, vl):
        res = _native.JobResult()
        _native.check(L.luda_build_from_sorted(keys.data_ptr(), klen, tr.data_ptr(), values.data_ptr(),
                                               voff.data_ptr(), vl.data_ptr(), n, 4096, 16, 10, sst_target,
                                               ctypes.byref(res), s.value))
        return res

    r_lo = build(tr_lo, voff_lo, vlen_lo)
    r_up = build(tr_up, voff_up, vlen_up)
    # arena: [pad][lower SSTs][pad][upper SSTs][pad]; files are byte-addressed (any alignment)
    pad = 4096
    size_lo, size_up = r_lo.out_bytes, r_up.out_bytes
    total = pad + size_lo + pad + size_up + pad
    arena = torch.zeros(total, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize(dev)
    _native.check(L.luda_memcpy_d2d_async(arena.data_ptr() + pad, r_lo.out, size_lo, s.value))
    _native.check(L.luda_memcpy_d2d_async(arena.data_ptr() + 2 * pad + size_lo, r_up.out, size_up, s.value))
    _native.check(L.luda_stream_sync(s.value))
    w = Workload()
    w.file_off = [pad + r_lo.sst_off[i] for i in range(r_lo.n_sst)] + \
                 [2 * pad + size_lo + r_up.sst_off[i] for i in range(r_up.n_sst)]
    w.file_len = [r_lo.sst_len[i] for i in range(r_lo.n_sst)] + [r_up.sst_len[i] for i in range(r_up.n_sst)]
    w.n_lower = r_lo.n_sst
    w.n_upper = r_up.n_sst
    w.arena = arena
    w.total = total
    w.s_in = size_lo + size_up
    w.n_in = 2 * n
    w.n_out_expected = int((~is_del).sum().item())
    w.v_out = w.n_out_expected * vlen
    w.key_len = klen + 8
    w.stream = s.value
    L.luda_job_release(ctypes.byref(r_lo))
    L.luda_job_release(ctypes.byref(r_up))
    # generator truth for the tests (user keys, value bytes, value offsets of the Li run, delete flags)
    w.truth = (keys, values, voff_lo, is_del) if keep_truth else None
    del values, keys, words, hi, lo, tr_up, tr_lo, voff_up, voff_lo, vlen_up, vlen_lo, is_del, idx
    torch.cuda.empty_cache()
    return w


def _d2h(L, dptr, n):
    buf = (ctypes.c_uint8 * n)()
    from paper_2004_03054_b200 import _native
    _native.check(L.luda_stage_out_async(ctypes.addressof(buf), dptr, n, None))
    _native.check(L.luda_stream_sync(None))
    return bytes(buf)


def plan_subcompaction(w, L, rank, world, n_keys, per_file=1):
    """The §8e plan with P = world ranges (weak scaling: one range per GPU).
    Host-cached SST metadata (footer + index block + first key of each local
    file) → samples → NCCL all-gather → splitters; returns this rank's range
    and the wall time of the plan (reported, not in the timed steps)."""
    import torch
    import torch.distributed as dist
    from paper_2004_03054_b200 import subcompact as SC
    base = w.arena.data_ptr()
    idx_keys, upper_first = [], []
    for i, (off, ln) in enumerate(zip(w.file_off, w.file_len)):
        foot = _d2h(L, base + off + ln - 24, 24)
        _, _, ioff, ilen, _ = SC.FOOTER.unpack(foot)
        blob = _d2h(L, base + off + ioff, ilen)
        fake = blob + SC.FOOTER.pack(0, 0, 0, ilen, 0)  # footer pointing at the index copy
        keys = SC.index_user_keys(fake)
        idx_keys.append(keys)
        if i >= w.n_lower:  # Li+1 file: smallest user key from the first entry of its first block
            head = _d2h(L, base + off, 64)
            pos = 0
            shared, pos = SC._varint(head, pos)
            unshared, pos = SC._varint(head, pos)
            _, pos = SC._varint(head, pos)
            upper_first.append(head[pos:pos + unshared][:unshared - 8])
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    local = []
    for keys in idx_keys:
        step = max(1, len(keys) // per_file)
        local += keys[::step][:per_file]
    nfiles = torch.tensor([len(w.file_off)], device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(nfiles, op=dist.ReduceOp.MAX)
    rows = int(nfiles.item()) * per_file
    samples = [k for g in SC.allgather_bytes(SC.encode_samples(local, rows), world) for k in SC.decode_samples(g)]
    bnd_rows = int(nfiles.item())
    gathered_b = SC.allgather_bytes(SC.encode_samples(upper_first, bnd_rows), world)
    boundaries = [k for g in gathered_b for k in SC.decode_samples(g)]
    first_of_rank = [SC.decode_samples(g)[0] for g in gathered_b]
    spl = SC.choose_splitters(samples, sorted(boundaries)[1:], world)
    rng = SC.ranges_from_splitters(spl)
    plan_ms = (time.perf_counter() - t0) * 1e3
    aligned = len(rng) == world and all(rng[r][0] == (None if r == 0 else first_of_rank[r]) for r in range(world))
    if aligned:
        lo, hi = rng[rank]
    else:  # ranges must match the locally held shard in this device-resident benchmark
        lo = None if rank == 0 else first_of_rank[rank]
        hi = None if rank == world - 1 else first_of_rank[rank + 1]
    return {"lo": lo, "hi": hi, "aligned": aligned, "plan_ms": plan_ms, "samples": len(samples),
            "splitters": len(spl)}


def set_range(desc, lo, hi):
    from paper_2004_03054_b200 import _native
    keep = []
    for name, key in (("range_lo", lo), ("range_hi", hi)):
        if key is not None:
            kb = (ctypes.c_uint8 * len(key)).from_buffer_copy(key)
            keep.append(kb)
            setattr(desc, name, ctypes.cast(kb, _native.c_u8p))
            setattr(desc, name + "_len", len(key))
    return keep


def job_desc(w, arena_ptr):
    from paper_2004_03054_b200 import _native
    n = len(w.file_off)
    fo = (ctypes.c_uint64 * n)(*w.file_off)
    fl = (ctypes.c_uint64 * n)(*w.file_len)
    rf = (ctypes.c_uint32 * 3)(0, w.n_lower, n)
    d = _native.JobDesc()
    d.arena = arena_ptr
    d.arena_bytes = w.total
    d.n_files = n
    d.file_off = ctypes.cast(fo, _native.c_u64p)
    d.file_len = ctypes.cast(fl, _native.c_u64p)
    d.n_runs = 2
    d.run_first_file = ctypes.cast(rf, _native.c_u32p)
    d.block_size, d.restart_interval, d.bits_per_key, d.sst_size_target = 4096, 16, 10, MIB4
    return d, (fo, fl, rf)


# --------------------------------------------------------------------------------------------
# CPU baseline (oracle port, bounded sample)
# --------------------------------------------------------------------------------------------
def _cpu_sample_job(n_keys, seed):
    from oracle import jobgen
    job = jobgen.c3(n=n_keys, seed=seed, sst_target=MIB4)
    lower, upper = jobgen.materialize(job)
    return lower + upper


_CPU_FILES = None


def _cpu_init(n_keys, seed):
    """Pool initializer: each worker builds its own c3-shaped input once (untimed)."""
    global _CPU_FILES
    import multiprocessing as mp
    ident = mp.current_process()._identity
    _CPU_FILES = _cpu_sample_job(n_keys, seed + (ident[0] if ident else 0))


def _cpu_compact(_):
    from oracle import luda_oracle as O
    t0 = time.perf_counter()
    O.reference_compact(_CPU_FILES)
    dt = time.perf_counter() - t0
    return sum(len(f) for f in _CPU_FILES), dt


def cpu_baseline(n_keys=1 << 19, workers=1, reps=1, seed=0xC3):
    """Oracle (pure-Python restatement of the reference, pinned to its golden
    outputs) on a bounded c3-shaped sample of 2 x n_keys entries; `workers`
    independent processes (one job each) = the host cores. Returns
    (MB/s, keys/s, seconds of the slowest worker)."""
    if workers <= 1:
        _cpu_init(n_keys, seed)
        b, dt = _cpu_compact(0)
        return b / dt / 1e6, 2 * n_keys / dt, dt
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_cpu_init, initargs=(n_keys, seed)) as pool:
        res = pool.map(_cpu_compact, range(workers), chunksize=1)
    t_max = max(r[1] for r in res)
    return sum(r[0] for r in res) / t_max / 1e6, 2 * n_keys * workers / t_max, t_max


def run_reference(args):
    """--impl reference: the reference algorithm (oracle port) on all host
    cores, one c3-shaped job per core built once; each step = one compaction
    per worker, throughput = bytes of all workers / slowest worker."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = len(os.sched_getaffinity(0))
    n_keys = args.cpu_keys
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    vals = []
    with ctx.Pool(cores, initializer=_cpu_init, initargs=(n_keys, 0xC3)) as pool:
        for i in range(args.warmup + args.steps):
            res = pool.map(_cpu_compact, range(cores), chunksize=1)
            t_max = max(r[1] for r in res)
            if i >= args.warmup:
                vals.append((sum(r[0] for r in res) / t_max / 1e6, 2 * n_keys * cores / t_max))
    mbps = statistics.median(v[0] for v in vals)
    keys_s = statistics.median(v[1] for v in vals)
    sample = f"c3-shaped job of 2x{n_keys} entries (16B/128B, 20% deletes) per worker, {cores} workers"
    out = {"impl": "reference", "metric": METRIC, "value": round(mbps, 3), "unit": "MB/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u8", "data": "synthetic",
           "config": {"workload": CONFIGS["c3"], "sample": sample},
           "keys_per_s": round(keys_s, 1),
           "cpu_baseline": {"value": round(mbps, 3), "unit": "MB/s", "cores": cores, "kind": "port",
                            "sample": sample},
           "e2e": {"value": round(mbps, 3), "unit": "MB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# --------------------------------------------------------------------------------------------
# main GPU arm
# --------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--keys", type=int, default=1 << 25, help="distinct keys per run (c3: 2^25 → 64M entries)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-keys", type=int, default=1 << 17,
                    help="reference arm: distinct keys per run of each worker's c3-shaped job")
    ap.add_argument("--cpu-baseline-keys", type=int, default=1 << 21,
                    help="cpu_baseline: distinct keys per run of the single-core c3-shaped sample (~10-30 s)")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; BENCH_DIST_BACKEND=gloo lets a multi-rank run share one GPU (functional test only)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2004_03054_b200 import _native
    L = _native.lib(local)
    w = synth_c3(args.keys, seed=0xC3 + 7919 * rank, device_index=local, shard=rank, nshards=world)
    desc, keep = job_desc(w, w.arena.data_ptr())
    st = w.stream
    plan = None
    if world > 1:
        # Subcompaction plan of the global job: index-key samples of the local files,
        # NCCL all-gather, splitters snapped to Li+1 file boundaries; this rank compacts range `rank`.
        plan = plan_subcompaction(w, L, rank, world, args.keys)
        keep = list(keep) + [set_range(desc, plan["lo"], plan["hi"])]

    def one_step():
        res = _native.JobResult()
        _native.check(L.luda_compact(ctypes.byref(desc), ctypes.byref(res), st))
        return res

    # correctness spot-check of the job shape
    res = one_step()
    assert res.n_in == w.n_in, (res.n_in, w.n_in)
    assert res.n_out == w.n_out_expected, (res.n_out, w.n_out_expected)
    s_out = res.out_bytes
    n_sst = res.n_sst
    L.luda_job_release(ctypes.byref(res))
    for _ in range(max(0, args.warmup - 1)):
        L.luda_job_release(ctypes.byref(one_step()))

    ev0, ev1 = ctypes.c_void_p(), ctypes.c_void_p()
    _native.check(L.luda_event_create(ctypes.byref(ev0)))
    _native.check(L.luda_event_create(ctypes.byref(ev1)))
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    k_acc = [0.0] * 8
    t_acc = [0.0] * 8
    launches = 0
    _native.check(L.luda_event_record(ev0.value, st))
    for _ in range(args.steps):
        r = one_step()
        for i in range(8):
            k_acc[i] += r.k_ms[i]
            t_acc[i] += r.t_ms[i]
        launches += r.launches
        L.luda_job_release(ctypes.byref(r))
    _native.check(L.luda_event_record(ev1.value, st))
    _native.check(L.luda_event_wait(ev1.value))
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = ctypes.c_float()
    _native.check(L.luda_event_elapsed_ms(ev0.value, ev1.value, ctypes.byref(ms)))
    t_step = ms.value / args.steps
    if world > 1:
        tt = torch.tensor([t_step], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.barrier()
        t_step = float(tt.item())

    # ---- e2e through the C ABI with host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        from paper_2004_03054_b200.device import PinnedBuffer
        pin_in, pin_out = PinnedBuffer(), PinnedBuffer()
        pin_in.ensure(w.total)
        pin_out.ensure(s_out + 4096)
        _native.check(L.luda_stage_out_async(pin_in.ptr, w.arena.data_ptr(), w.total, st))
        _native.check(L.luda_stream_sync(st))
        # Two input arenas: the H2D of step i+1 (in_lower / in_upper streams) runs while step i compacts and
        # step i-1's output streams back (out stream) — PCIe is full duplex, so a step costs ~max(H2D, D2H+job).
        arenas = [torch.empty(w.total, dtype=torch.uint8, device="cuda") for _ in range(2)]
        descs = []
        for ar in arenas:
            d2, k2 = job_desc(w, ar.data_ptr())
            if plan is not None:
                k2 = list(k2) + [set_range(d2, plan["lo"], plan["hi"])]
            descs.append((d2, k2))
        pin_out2 = PinnedBuffer()
        pin_out2.ensure(s_out + 4096)
        pins_out = [pin_out, pin_out2]
        s_lo, s_up, s_o = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        for sp in (s_lo, s_up, s_o):
            _native.check(L.luda_stream_create(ctypes.byref(sp)))
        split = w.file_off[w.n_lower] if w.n_lower < len(w.file_off) else w.total
        ev_in = [[ctypes.c_void_p() for _ in range(2)] for _ in range(2)]
        ev_out = [ctypes.c_void_p() for _ in range(2)]
        e_c = ctypes.c_void_p()
        for e in [x for row in ev_in for x in row] + ev_out + [e_c]:
            _native.check(L.luda_event_create(ctypes.byref(e)))

        def stage(i):
            ar = arenas[i % 2]
            _native.check(L.luda_stage_in_async(ar.data_ptr(), pin_in.ptr, split, s_lo.value))
            _native.check(L.luda_stage_in_async(ar.data_ptr() + split, pin_in.ptr + split, w.total - split,
                                                s_up.value))
            _native.check(L.luda_event_record(ev_in[i % 2][0].value, s_lo.value))
            _native.check(L.luda_event_record(ev_in[i % 2][1].value, s_up.value))

        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        out_bytes = 0
        prev = None
        stage(0)
        for i in range(args.e2e_steps):
            if i + 1 < args.e2e_steps:
                stage(i + 1)  # arena (i+1)%2 was last read by job i-1, which has completed
            for e in ev_in[i % 2]:
                _native.check(L.luda_stream_wait_event(st, e.value))
            res = _native.JobResult()
            _native.check(L.luda_compact(ctypes.byref(descs[i % 2][0]), ctypes.byref(res), st))
            _native.check(L.luda_event_record(e_c.value, st))
            _native.check(L.luda_stream_wait_event(s_o.value, e_c.value))
            _native.check(L.luda_stage_out_async(pins_out[i % 2].ptr, res.out, res.out_bytes, s_o.value))
            _native.check(L.luda_event_record(ev_out[i % 2].value, s_o.value))
            out_bytes = res.out_bytes
            if prev is not None:  # step i-1's output buffer is recycled once its D2H has landed
                _native.check(L.luda_event_wait(ev_out[(i - 1) % 2].value))
                L.luda_job_release(ctypes.byref(prev))
            prev = res
        _native.check(L.luda_stream_sync(s_o.value))
        if prev is not None:
            L.luda_job_release(ctypes.byref(prev))
        dt = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            tt = torch.tensor([dt], device="cuda" if backend == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        e2e = {"value": round(world * w.s_in / dt / 1e6, 3), "unit": "MB/s", "h2d_bytes_per_step": w.total,
               "d2h_bytes_per_step": int(out_bytes), "ms_per_step": round(dt * 1e3, 3),
               "timing": "host wall clock over the steps: every step H2Ds its whole input from pinned host memory "
                         "(double-buffered arenas: step i+1's H2D overlaps step i's job and step i-1's D2H) and "
                         "D2Hs its whole output; all transfers complete inside the timed region"}
        pin_out2.free()
        pin_in.free()
        pin_out.free()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    peaks, peak_kind = load_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    K = w.key_len
    rec = K + 8
    s_in, n_in, n_out, v_out = w.s_in, w.n_in, w.n_out_expected, w.v_out
    b_alg = s_in + s_out + 2 * rec * (n_in + n_out) + v_out
    kms = [x / args.steps for x in k_acc]
    tms = [x / args.steps for x in t_acc]
    # algorithmic bytes per kernel launch
    kern = {
        "decode": (s_in + rec * n_in, kms[0]),
        "merge_resolve": (rec * n_in + rec * n_out, kms[1]),
        "block_plan": (rec * n_out + 8 * n_out, kms[2]),
        "encode": (rec * n_out + v_out + s_out, kms[3]),
        "sst_meta": (rec * n_out, kms[4]),
    }
    kernels = {k: {"alg_bytes": b, "ms": round(t, 4), "gbs": round(b / (t * 1e-3) / 1e9, 1) if t else None}
               for k, (b, t) in kern.items()}
    dom = max(kern, key=lambda k: kern[k][1])
    db, dt_ = kern[dom]
    ach = db / (dt_ * 1e-3) / 1e9
    traffic, traffic_src = None, None
    try:  # measured DRAM bytes per launch of that kernel (one ncu --set full capture, profiles/traffic.json)
        tj = json.load(open(os.path.join(REPO, "profiles", "traffic.json")))
        kname = {"decode": "decode_kernel", "merge_resolve": "merge_kernel", "encode": "encode_kernel",
                 "sst_meta": "sst_meta_kernel", "block_plan": "block_jump_kernel"}[dom]
        if kname in tj:
            traffic, traffic_src = tj[kname]["dram_bytes"], tj[kname]["source"]
    except Exception:
        pass
    cpu = None
    if not args.no_cpu and world == 1 or (not args.no_cpu and rank == 0):
        mbps, keys_s, wall = cpu_baseline(n_keys=args.cpu_baseline_keys, workers=1)
        cpu = {"value": round(mbps, 4), "unit": "MB/s", "cores": 1, "kind": "port",
               "sample": f"oracle (the reference algorithm restated in Python+zlib+numpy, pinned to the reference's "
                         f"golden outputs) on a c3-shaped job of 2x{args.cpu_baseline_keys} entries (16B/128B, "
                         f"20% deletes): {wall:.1f}s of compaction", "keys_per_s": round(keys_s, 1)}
    value = world * s_in / (t_step * 1e-3) / 1e6
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "MB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": workload_text(args.keys, world), "keys_per_run": args.keys, "n_in": n_in, "n_out": n_out,
                   "input_bytes": s_in, "output_bytes": int(s_out), "input_ssts": len(w.file_off),
                   "output_ssts": int(n_sst), "block_size": 4096, "sst_size_target": MIB4,
                   "l2": "inputs (%.1f GB) larger than L2; no flush" % (s_in / 1e9),
                   "parallelism": f"key-range subcompactions x{world}" if world > 1 else "1 GPU",
                   "subcompaction_plan": None if plan is None else {
                       k: (v.hex() if isinstance(v, bytes) else v) for k, v in plan.items()}},
        "keys_per_s": round(world * n_in / (t_step * 1e-3), 1),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(ach / hbm, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind,
                     "alg_bytes_per_launch": db},
        "job_roofline": {"alg_bytes": b_alg, "achieved": round(b_alg / (t_step * 1e-3) / 1e9, 1), "peak": hbm,
                         "frac": round(b_alg / (t_step * 1e-3) / 1e9 / hbm, 4),
                         "formula": "S_in + S_out + 2(K+8)(N_in+N_out) + V_out"},
        "kernels": kernels,
        "phases_ms": {"parse": round(tms[0], 3), "decode": round(tms[1], 3), "merge": round(tms[2], 3),
                      "plan": round(tms[3], 3), "emit": round(tms[4], 3), "total": round(tms[7], 3)},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
