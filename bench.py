"""LUDA compaction benchmark on B200 (BASELINE.json metric: compaction input
MB/s and keys/s per B200 at 1/2/4/8 GPUs; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--extras c2,c4,reads,storage,c5]

N = 1 (headline): a step = one full compaction job of BASELINE config 3
(luda_compact: parse → decode → merge/resolve → plan → encode →
filter/index/footer) over 2 × 2^25 entries (9.6 GB of input SSTs, far larger
than L2 — no flush needed between steps).
  * value : device-resident (inputs in HBM when the timed region starts,
            outputs left in HBM), CUDA events on the job's stream;
  * e2e   : the same job through the C ABI with HOST buffers — pinned H2D of
            every input on the in_lower / in_upper streams, the job, D2H of
            every output — double-buffered across steps, host wall clock;
  * workloads: the other BASELINE configs measured in the same run — c2
            latency (1 L1 + 10 L2 x 2 MB, p50/p99 over 100 jobs), c4 scaled
            (8 overlapping L0 runs x 2^22 24-byte keys), c5 on 1 GPU (the
            strong-scaling base of the multi-GPU line).
N > 1 (torchrun, or `--gpus N` which re-executes itself under torchrun): the
line is BASELINE config 5 — ONE global ~256 GB job (bench_c5.py), P = 64
key ranges fixed for every N, splitters from the NCCL all-gather of index
samples, ranges dealt contiguously, each rank compacting its ranges in
waves synthesised on its device; strong scaling, max over ranks.
Inputs are synthesised on the GPU with this package's own SST builder (the
bytes equal SstBuilder's; tests/test_gpu_parity.py).
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

METRIC = "compaction input MB/s"
MIB4 = 4 * 2**20
C3_TEXT = ("Overwrite-heavy compaction: 64M KV pairs, 50% duplicate keys across runs plus 10% tombstones, "
           "16B/128B, 1 B200")
C5_TEXT = ("Key-range-partitioned bulk compaction of ~256GB synthetic input across 1/2/4/8 B200 "
           "(subcompaction splitter all-gather over NCCL)")


def c3_text(keys):
    t = C3_TEXT
    if keys != 1 << 25:
        t = t.replace("64M KV pairs", f"{2 * keys / 2**20:g}M KV pairs (c3-shaped, reduced from 64M)")
    return t


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


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
        self.t = None

    def start(self, wait_s=3.0):
        """Start sampling and wait for the first sample (nvidia-smi needs ~1 s
        to start; a short timed region would otherwise see no sample)."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
            return
        t0 = time.time()
        while not self.lines and time.time() - t0 < wait_s:
            time.sleep(0.02)
        self.mark = len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines[max(0, getattr(self, "mark", 0) - 1):]
        for ln in lines:
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
# GPU workload synthesis: sorted runs of SSTs built on the device
# --------------------------------------------------------------------------------------------
class Workload:
    pass


def synth_c3(n_keys, seed, device_index, del_frac=0.2, vlen=128, klen=16, sst_target=MIB4, keep_truth=False):
    """BASELINE c3 on the device: n_keys distinct 16-byte keys; Li+1 = every
    key (seq 1..n, Put, 128-byte values), Li = the same keys (newer seqs),
    del_frac of them Deletes; both runs cut into 4 MiB SSTs by the device
    builder and laid out in one arena."""
    import torch

    from paper_2004_03054_b200 import _native
    L = _native.lib(device_index)
    dev = torch.device("cuda", device_index)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    n = n_keys
    # sorted distinct 16-byte keys: sorted random 64-bit prefix (sign-flipped → unsigned order) + random suffix
    while True:
        hi = torch.randint(-2**63, 2**63 - 1, (n,), generator=g, device=dev, dtype=torch.int64)
        hi, _ = torch.sort(hi)
        if bool((hi[1:] != hi[:-1]).all()):
            break
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


def synth_c4(L, runs, n, seed, stream, klen=24, vlen=256):
    """BASELINE c4 (scaled): `runs` L0 files, each a sorted run of n uniform
    24-byte keys with 256-byte values, file i newer than file i+1, each built
    as ONE SST (sst_size_target 2^31, under the u32 4 GiB cap) by the device
    builder. Returns (arena tensor, file offsets, file lengths)."""
    import torch
    from paper_2004_03054_b200 import _native
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    values = torch.empty(n * vlen + 4096, dtype=torch.uint8, device=dev).random_(0, 256, generator=g)
    idx = torch.arange(n, device=dev, dtype=torch.int64)
    voff = idx * vlen
    vl = torch.full((n,), vlen, dtype=torch.int32, device=dev)
    outs = []
    for r in range(runs):
        while True:
            hi = torch.randint(-2**63, 2**63 - 1, (n,), generator=g, device=dev, dtype=torch.int64)
            hi, _ = torch.sort(hi)
            if bool((hi[1:] != hi[:-1]).all()):
                break
        hi = hi ^ torch.tensor(-2**63, dtype=torch.int64, device=dev)  # signed order -> unsigned byte order
        rest = [torch.randint(-2**63, 2**63 - 1, (n,), generator=g, device=dev, dtype=torch.int64)
                for _ in range((klen - 8) // 8)]
        words = torch.stack([hi] + rest, 1).contiguous()
        keys = words.view(torch.uint8).view(n, klen // 8, 8).flip(2).reshape(n * klen).contiguous()
        seq0 = (runs - 1 - r) * n  # file 0 is the newest
        tr = ((idx + seq0 + 1) << 8) | 1
        torch.cuda.synchronize(dev)
        res = _native.JobResult()
        _native.check(L.luda_build_from_sorted(keys.data_ptr(), klen, tr.data_ptr(), values.data_ptr(),
                                               voff.data_ptr(), vl.data_ptr(), n, 4096, 16, 10, 1 << 31,
                                               ctypes.byref(res), stream))
        assert res.n_sst == 1
        outs.append(res)
    total = sum(r.out_bytes for r in outs)
    arena = torch.zeros(total + 4096, dtype=torch.uint8, device=dev)
    offs, lens, at = [], [], 0
    for r in outs:
        _native.check(L.luda_memcpy_d2d_async(arena.data_ptr() + at, r.out, r.out_bytes, stream))
        offs.append(at)
        lens.append(r.out_bytes)
        at += r.out_bytes
    _native.check(L.luda_stream_sync(stream))
    for r in outs:
        L.luda_job_release(ctypes.byref(r))
    return arena, offs, lens


def synth_c2(L, stream, seed=0xC2, n_upper=19640, n_lower=1964, vlen=1024, upper_file_keys=1964):
    """BASELINE c2: 10 L2 SSTs of ~2 MB (one run of n_upper keys, a file
    every upper_file_keys entries) and 1 L1 SST of n_lower keys spread
    uniformly over the same key space (newer); 16-byte keys, 1 KB values.
    Returns (arena, offs, lens, n_lower_files)."""
    import torch
    from paper_2004_03054_b200 import _native
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    n = n_upper + n_lower
    while True:
        hi = torch.randint(-2**63, 2**63 - 1, (n,), generator=g, device=dev, dtype=torch.int64)
        hi, _ = torch.sort(hi)
        if bool((hi[1:] != hi[:-1]).all()):
            break
    hi = hi ^ torch.tensor(-2**63, dtype=torch.int64, device=dev)
    lo = torch.randint(-2**63, 2**63 - 1, (n,), generator=g, device=dev, dtype=torch.int64)
    is_low = torch.zeros(n, dtype=torch.bool, device=dev)
    is_low[torch.randperm(n, generator=g, device=dev)[:n_lower]] = True
    values = torch.empty(n * vlen + 4096, dtype=torch.uint8, device=dev).random_(0, 256, generator=g)
    parts = []
    for sel, seq0, fk in ((is_low, n_upper, 0), (~is_low, 0, upper_file_keys)):
        ids = torch.nonzero(sel).flatten()
        m = ids.numel()
        words = torch.stack([hi[ids], lo[ids]], 1).contiguous()
        keys = words.view(torch.uint8).view(m, 2, 8).flip(2).reshape(m * 16).contiguous()
        tr = ((torch.arange(m, device=dev, dtype=torch.int64) + seq0 + 1) << 8) | 1
        voff = ids * vlen
        vl = torch.full((m,), vlen, dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)
        res = _native.JobResult()
        _native.check(L.luda_build_files_from_sorted(keys.data_ptr(), 16, tr.data_ptr(), values.data_ptr(),
                                                     voff.data_ptr(), vl.data_ptr(), m, 4096, 16, 10, 1 << 31, fk,
                                                     ctypes.byref(res), stream))
        parts.append(res)
    total = sum(r.out_bytes for r in parts) + 4096
    arena = torch.zeros(total, dtype=torch.uint8, device=dev)
    offs, lens, at = [], [], 0
    for r in parts:
        _native.check(L.luda_memcpy_d2d_async(arena.data_ptr() + at, r.out, r.out_bytes, stream))
        offs += [at + r.sst_off[i] for i in range(r.n_sst)]
        lens += [r.sst_len[i] for i in range(r.n_sst)]
        at += r.out_bytes
    _native.check(L.luda_stream_sync(stream))
    n_low_files = parts[0].n_sst
    for r in parts:
        L.luda_job_release(ctypes.byref(r))
    return arena, offs, lens, n_low_files


def make_desc(arena_ptr, arena_bytes, offs, lens, run_first, sst_target=MIB4, lo=None, hi=None):
    """luda_job_desc over files in one device arena; returns (desc, keep-alive)."""
    from paper_2004_03054_b200 import _native
    n = len(offs)
    fo = (ctypes.c_uint64 * max(n, 1))(*offs)
    fl = (ctypes.c_uint64 * max(n, 1))(*lens)
    rf = (ctypes.c_uint32 * len(run_first))(*run_first)
    d = _native.JobDesc()
    d.arena, d.arena_bytes, d.n_files = arena_ptr, arena_bytes, n
    d.file_off = ctypes.cast(fo, _native.c_u64p)
    d.file_len = ctypes.cast(fl, _native.c_u64p)
    d.n_runs = len(run_first) - 1
    d.run_first_file = ctypes.cast(rf, _native.c_u32p)
    d.block_size, d.restart_interval, d.bits_per_key, d.sst_size_target = 4096, 16, 10, sst_target
    keep = [fo, fl, rf]
    for name, key in (("range_lo", lo), ("range_hi", hi)):
        if key is not None:
            kb = (ctypes.c_uint8 * len(key)).from_buffer_copy(key)
            keep.append(kb)
            setattr(d, name, ctypes.cast(kb, _native.c_u8p))
            setattr(d, name + "_len", len(key))
    return d, keep


def job_desc(w, arena_ptr):
    return make_desc(arena_ptr, w.total, w.file_off, w.file_len, [0, w.n_lower, len(w.file_off)])


class Timer:
    """CUDA events on a stream (the jobs' stream: torch's events only see torch's current stream)."""

    def __init__(self, L):
        from paper_2004_03054_b200 import _native
        self.L, self.N = L, _native
        self.a, self.b = ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(L.luda_event_create(ctypes.byref(self.a)))
        _native.check(L.luda_event_create(ctypes.byref(self.b)))

    def start(self, st):
        self.N.check(self.L.luda_event_record(self.a.value, st))

    def stop(self, st):
        self.N.check(self.L.luda_event_record(self.b.value, st))
        self.N.check(self.L.luda_event_wait(self.b.value))
        ms = ctypes.c_float()
        self.N.check(self.L.luda_event_elapsed_ms(self.a.value, self.b.value, ctypes.byref(ms)))
        return ms.value


def e2e_public_api(w, steps):
    """c3 end to end through the package's public API: ``run_compactions``
    over `steps` copies of the job, inputs in pinned host memory
    (``StagedInput``, filled from the device arena once, untimed). Every step
    H2Ds its whole input and D2Hs its whole output inside the timed region
    (double-buffered: step k+1's H2D overlaps step k's job and step k-1's
    D2H). Host wall clock."""
    from paper_2004_03054_b200 import DeviceConfig, _native, make_device, run_compactions
    from paper_2004_03054_b200.compaction import StagedInput
    from paper_2004_03054_b200.version import CompactionJob, SstMeta, Version
    L = _native.lib(0)
    dev = make_device(DeviceConfig(backend="b200"))
    staged = StagedInput(w.file_len)
    for i, (o, ln) in enumerate(zip(w.file_off, w.file_len)):
        _native.check(L.luda_stage_out_async(staged.buf.ptr + staged.offs[i], w.arena.data_ptr() + o, ln, w.stream))
    _native.check(L.luda_stream_sync(w.stream))
    metas = [SstMeta(file_id=i + 1, file_size=ln, smallest=b"", largest=b"", level=1 if i < w.n_lower else 2)
             for i, ln in enumerate(w.file_len)]
    job = CompactionJob(source_level=1, lower=metas[:w.n_lower], upper=metas[w.n_lower:], target_level=2,
                        version=Version.empty())
    # two untimed jobs: grow BOTH double-buffer slots (device arena + pinned output buffer of each)
    for outs, st in run_compactions([(job, staged)] * 2, dev):
        pass
    t0 = time.perf_counter()
    out_bytes, n_out = 0, 0
    for outs, st in run_compactions([(job, staged)] * steps, dev):
        out_bytes = sum(len(d) for d, _ in outs)
        n_out = st.n_out
    dt = (time.perf_counter() - t0) / steps
    assert n_out == w.n_out_expected
    staged.free()
    dev.close()
    return {"value": round(w.s_in / dt / 1e6, 3), "unit": "MB/s", "h2d_bytes_per_step": staged.total,
            "d2h_bytes_per_step": int(out_bytes), "ms_per_step": round(dt * 1e3, 3),
            "api": "paper_2004_03054_b200.run_compactions (StagedInput pinned inputs, memoryview outputs)",
            "timing": "host wall clock over the steps: every step H2Ds its whole input from pinned host memory "
                      "and D2Hs its whole output (double-buffered pipeline: step k+1's H2D overlaps step k's job "
                      "and step k-1's D2H); all transfers complete inside the timed region"}


def compact_once(L, desc, st):
    from paper_2004_03054_b200 import _native
    res = _native.JobResult()
    _native.check(L.luda_compact(ctypes.byref(desc), ctypes.byref(res), st))
    return res


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(round(q / 100 * (len(xs) - 1))))]


# --------------------------------------------------------------------------------------------
# other BASELINE configs at N = 1
# --------------------------------------------------------------------------------------------
def measure_c2(L, stream, jobs=100, warmup=5):
    """c2 latency: device time (events) and host wall time per job, plus the
    end-to-end job (pinned H2D of the inputs, job, D2H of the outputs)."""
    from paper_2004_03054_b200 import _native
    from paper_2004_03054_b200.device import PinnedBuffer
    arena, offs, lens, nlow = synth_c2(L, stream)
    total = offs[-1] + lens[-1]
    desc, keep = make_desc(arena.data_ptr(), total, offs, lens, [0, nlow, len(offs)])
    tm = Timer(L)
    dev_ms, wall_ms = [], []
    out_b = 0
    for i in range(warmup + jobs):
        t0 = time.perf_counter()
        tm.start(stream)
        res = compact_once(L, desc, stream)
        ms = tm.stop(stream)
        w = (time.perf_counter() - t0) * 1e3
        out_b, nsst, n_in, n_out, launches = res.out_bytes, res.n_sst, res.n_in, res.n_out, res.launches
        L.luda_job_release(ctypes.byref(res))
        if i >= warmup:
            dev_ms.append(ms)
            wall_ms.append(w)
    # end to end through the C ABI with host buffers
    pin_in, pin_out = PinnedBuffer(), PinnedBuffer()
    pin_in.ensure(total)
    pin_out.ensure(out_b + 4096)
    _native.check(L.luda_stage_out_async(pin_in.ptr, arena.data_ptr(), total, stream))
    _native.check(L.luda_stream_sync(stream))
    import torch
    ar2 = torch.empty(total + 4096, dtype=torch.uint8, device=arena.device)
    desc2, keep2 = make_desc(ar2.data_ptr(), total, offs, lens, [0, nlow, len(offs)])
    e2e_ms = []
    for i in range(warmup + jobs // 2):
        t0 = time.perf_counter()
        _native.check(L.luda_stage_in_async(ar2.data_ptr(), pin_in.ptr, total, stream))
        res = compact_once(L, desc2, stream)
        _native.check(L.luda_stage_out_async(pin_out.ptr, res.out, res.out_bytes, stream))
        _native.check(L.luda_stream_sync(stream))
        L.luda_job_release(ctypes.byref(res))
        if i >= warmup:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    pin_in.free()
    pin_out.free()
    return {"workload": "L1->L2 compaction: 1 L1 SST vs 10 overlapping L2 SSTs, 2MB each, 16B keys / 1KB values, "
                        "1 B200 (BASELINE config 2)",
            "input_bytes": total, "input_ssts": len(offs), "output_ssts": nsst, "n_in": n_in, "n_out": n_out,
            "jobs": jobs, "device_ms_p50": round(pct(dev_ms, 50), 4), "device_ms_p99": round(pct(dev_ms, 99), 4),
            "host_ms_p50": round(pct(wall_ms, 50), 4), "host_ms_p99": round(pct(wall_ms, 99), 4),
            "e2e_ms_p50": round(pct(e2e_ms, 50), 4), "e2e_ms_p99": round(pct(e2e_ms, 99), 4),
            "mb_s_device_p50": round(total / (pct(dev_ms, 50) * 1e-3) / 1e6, 1),
            "launches_per_job": launches,
            "note": "latency-bound (roofline time ~11 us): device_ms = CUDA events around luda_compact on its "
                    "stream; host_ms = the same call's host wall time (includes host orchestration); e2e_ms = "
                    "pinned H2D of the 23 MB input + job + D2H of the outputs"}


def measure_c4(L, stream, steps=5, warmup=2, n=1 << 22, peak=6539.5):
    arena, offs, lens = synth_c4(L, 8, n, 0xC4, stream)
    desc, keep = make_desc(arena.data_ptr(), arena.numel(), offs, lens, list(range(9)))
    tm = Timer(L)
    ms = []
    for i in range(warmup + steps):
        tm.start(stream)
        res = compact_once(L, desc, stream)
        t = tm.stop(stream)
        s_out, n_in, n_out, kms = res.out_bytes, res.n_in, res.n_out, list(res.k_ms)
        L.luda_job_release(ctypes.byref(res))
        if i >= warmup:
            ms.append(t)
    t = statistics.median(ms)
    s_in = sum(lens)
    rec = 24 + 8 + 8
    b_alg = s_in + s_out + 2 * rec * (n_in + n_out) + n_out * 256
    return {"workload": "Unsorted-L0 stress: 8 overlapping L0 files with random keys, 24B keys / 256B values "
                        f"(BASELINE config 4, scaled: 8 x {n} keys, one SST per file)",
            "input_bytes": s_in, "n_in": n_in, "n_out": n_out, "ms_per_job": round(t, 3),
            "value": round(s_in / (t * 1e-3) / 1e6, 1), "unit": "MB/s", "keys_per_s": round(n_in / (t * 1e-3), 1),
            "job_roofline": {"alg_bytes": b_alg, "frac": round(b_alg / (t * 1e-3) / 1e9 / peak, 4)},
            "kernel_ms": {"decode": round(kms[0], 3), "merge_final": round(kms[1], 3), "encode": round(kms[3], 3),
                          "sst_meta": round(kms[4], 3)}}


def measure_reads(L, desc, st, n_lookups=1 << 22, steps=10, warmup=3):
    """Batched point lookups over the c3 job's output SSTs,
    opened in place in HBM (987 x 4 MiB SSTs, 26.8M entries): half the keys
    present (index keys of the outputs), half absent random 16 B keys, probed
    in store order over the one output level (range binary search → bloom →
    index → block). Device: the lookup kernel alone over device-resident keys
    (CUDA events). e2e: luda_tables_get with host keys (H2D keys, lookups,
    packing, D2H of the found keys and values)."""
    import random
    import struct as _st

    import torch
    from paper_2004_03054_b200 import _native
    res = compact_once(L, desc, st)
    try:
        n_sst = res.n_sst
        offs = [res.sst_off[i] for i in range(n_sst)]
        lens = [res.sst_len[i] for i in range(n_sst)]
        # present keys: the outputs' index keys (last key of every block), read back from the device
        foot = (ctypes.c_uint8 * 24)()
        present = []
        for i in range(n_sst):
            _native.check(L.luda_stage_out_async(foot, res.out + offs[i] + lens[i] - 24, 24, st))
            _native.check(L.luda_stream_sync(st))
            _, _, ioff, ilen, _ = _st.unpack("<IIIIQ", bytes(foot))
            ib = (ctypes.c_uint8 * ilen)()
            _native.check(L.luda_stage_out_async(ib, res.out + offs[i] + ioff, ilen, st))
            _native.check(L.luda_stream_sync(st))
            b = bytes(ib)
            p = 0
            while p < ilen - 8:
                kl = b[p]
                present.append(b[p + 1:p + 1 + kl - 8])
                p += 1 + kl + 8
        rng = random.Random(0x7EAD)
        keys = [rng.choice(present) if i % 2 == 0 else rng.randbytes(16) for i in range(n_lookups)]
        blob = b"".join(keys)
        h = ctypes.c_void_p()
        off_arr = (ctypes.c_uint64 * n_sst)(*offs)
        len_arr = (ctypes.c_uint64 * n_sst)(*lens)
        t0 = time.perf_counter()
        _native.check(L.luda_tables_open(res.out, off_arr, len_arr, n_sst, ctypes.byref(h), st))
        open_ms = (time.perf_counter() - t0) * 1e3
        sk = _native.sst_key_pairs(res)
        rk = b"".join(a[:-8] + b[:-8] for a, b in sk)
        rl = [x for a, b in sk for x in (len(a) - 8, len(b) - 8)]
        plan = _native.ProbePlan(0, None, 1, (ctypes.c_uint32 * 2)(0, n_sst),
                                 (ctypes.c_uint32 * n_sst)(*range(n_sst)),
                                 (ctypes.c_uint8 * len(rk)).from_buffer_copy(rk), (ctypes.c_uint32 * len(rl))(*rl))
        _native.check(L.luda_tables_set_plan(h.value, ctypes.byref(plan), st))
        dk = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda()
        dko = (torch.arange(n_lookups, dtype=torch.int64) * 16).cuda()
        dkl = torch.full((n_lookups,), 16, dtype=torch.int32).cuda()
        torch.cuda.synchronize()
        for _ in range(warmup):
            _native.check(L.luda_tables_lookup_dev(h.value, dk.data_ptr(), dko.data_ptr(), dkl.data_ptr(),
                                                   n_lookups, None, 256, st))
        tm = Timer(L)
        tm.start(st)
        for _ in range(steps):
            _native.check(L.luda_tables_lookup_dev(h.value, dk.data_ptr(), dko.data_ptr(), dkl.data_ptr(),
                                                   n_lookups, None, 256, st))
        ms = tm.stop(st) / steps
        # e2e through the C ABI with host keys (pinned, fixed 16-byte keys back to back)
        from paper_2004_03054_b200.device import PinnedBuffer
        pk = PinnedBuffer()
        pk.ensure(len(blob))
        ctypes.memmove(pk.ptr, blob, len(blob))
        kl = (ctypes.c_uint32 * 1)(16)
        r = _native.GetResult()
        kptr = ctypes.cast(pk.ptr, _native.c_u8p)
        _native.check(L.luda_tables_get(h.value, kptr, len(blob), None, kl, n_lookups, None, 256, ctypes.byref(r), st))
        e2e = []
        for _ in range(3):
            t0 = time.perf_counter()
            _native.check(L.luda_tables_get(h.value, kptr, len(blob), None, kl, n_lookups, None, 256,
                                            ctypes.byref(r), st))
            e2e.append(time.perf_counter() - t0)
        found = sum(1 for i in range(n_lookups) if r.status[i] == 1)
        pk.free()
        e2e_s = min(e2e)
        out = {"workload": "Batched point lookups (Table.get in store order) over the c3 job's %d output SSTs "
                           "resident in HBM: %d keys, 50%% present / 50%% absent" % (n_sst, n_lookups),
               "lookups": n_lookups, "found": found, "ms": round(ms, 3),
               "value": round(n_lookups / (ms * 1e-3), 1), "unit": "lookups/s", "open_ms": round(open_ms, 2),
               "e2e": {"value": round(n_lookups / e2e_s, 1), "unit": "lookups/s", "ms": round(e2e_s * 1e3, 2),
                       "h2d_bytes": len(blob) + 4, "d2h_bytes": int(r.packed_bytes) + 40 * n_lookups,
                       "t_ms": [round(x, 3) for x in r.t_ms]}}
        L.luda_tables_close(h.value)
        return out
    finally:
        L.luda_job_release(ctypes.byref(res))


def measure_storage(L, w, st, steps=2, root="/tmp/luda_bench_io"):
    """Storage → HBM → storage: the c3 job's 2,261 input SSTs read from files
    straight into the device arena (luda_files_read), compacted, and the 987
    output SSTs written from device memory to files (luda_files_write) —
    SURVEY §8f row 3. cuFile is used when the host supports GPUDirect Storage
    (LUDA_GDS=1), else the native 8-thread pread/pwrite ↔ pinned ↔ H2D/D2H
    pipeline. The input files are written once, untimed (they sit in the page
    cache: the number is the I/O-path ceiling, not a cold-disk figure)."""
    import shutil

    import torch
    from paper_2004_03054_b200 import _native
    shutil.rmtree(root, ignore_errors=True)
    os.makedirs(os.path.join(root, "in"))
    os.makedirs(os.path.join(root, "out"))
    try:
        n = len(w.file_off)
        paths = (ctypes.c_char_p * n)(*[os.path.join(root, "in", f"{i}.sst").encode() for i in range(n)])
        fo = (ctypes.c_uint64 * n)(*w.file_off)
        fl = (ctypes.c_uint64 * n)(*w.file_len)
        used = ctypes.c_int()
        _native.check(L.luda_files_write(paths, n, w.arena.data_ptr(), fo, fl, 0, ctypes.byref(used)))
        arena = torch.empty(w.total, dtype=torch.uint8, device="cuda")
        desc, keep = job_desc(w, arena.data_ptr())
        torch.cuda.synchronize()
        t_in, t_job, t_out, out_b = [], [], [], 0
        for _ in range(steps):
            t0 = time.perf_counter()
            _native.check(L.luda_files_read(paths, n, arena.data_ptr(), fo, fl, 0, ctypes.byref(used)))
            t1 = time.perf_counter()
            res = compact_once(L, desc, st)
            _native.check(L.luda_stream_sync(st))
            t2 = time.perf_counter()
            m = res.n_sst
            op = (ctypes.c_char_p * m)(*[os.path.join(root, "out", f"{i}.sst").encode() for i in range(m)])
            _native.check(L.luda_files_write(op, m, res.out, res.sst_off, res.sst_len, 0, ctypes.byref(used)))
            t3 = time.perf_counter()
            out_b = res.out_bytes
            L.luda_job_release(ctypes.byref(res))
            t_in.append(t1 - t0)
            t_job.append(t2 - t1)
            t_out.append(t3 - t2)
        tot = min(a + b + c for a, b, c in zip(t_in, t_job, t_out))
        return {"workload": "c3 job storage -> HBM -> storage (%d input files, %d outputs)" % (n, m),
                "path": {1: "cuFile (GPUDirect Storage)", 2: "native pread/pwrite <-> pinned <-> H2D/D2H, 8 threads"
                         }[used.value],
                "value": round(w.s_in / tot / 1e6, 1), "unit": "MB/s", "s_per_step": round(tot, 3),
                "read_GBps": round(w.s_in / min(t_in) / 1e9, 2), "write_GBps": round(out_b / min(t_out) / 1e9, 2),
                "job_ms": round(min(t_job) * 1e3, 2), "input_bytes": w.s_in, "output_bytes": int(out_b),
                "note": "input files in the page cache (written untimed just before)"}
    finally:
        shutil.rmtree(root, ignore_errors=True)


def measure_c5(world, rank, local, steps, warmup, group=None, total_gb=256.0):
    import bench_c5
    spec = bench_c5.C5Spec(total_gb=total_gb)
    tot = bench_c5.run(spec, local, world, rank, group=group, steps=steps, warmup=warmup)
    return spec, tot


# --------------------------------------------------------------------------------------------
# reference arm / CPU baseline
# --------------------------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the reference's own CPU compaction (bench_ref.py) on
    all host cores, each worker compacting a bounded sample of this arm's
    workload; rank 0 alone under torchrun."""
    import bench_ref
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", "1"))
    shape = "c3" if world == 1 else "c5"
    cores = len(os.sched_getaffinity(0))
    mbps, keys_s, kind, secs = bench_ref.inline_throughput(shape, args.cpu_keys, cores, args.steps,
                                                           args.warmup)
    sample = (f"{shape}-shaped job ({2 * args.cpu_keys if shape == 'c3' else args.cpu_keys + args.cpu_keys // 9} "
              f"entries, 16B/128B, 4 MiB SSTs) per worker, {cores} workers (one process per host core); "
              f"reference = the pip-installed /root/reference (baseline/_ref) composed per SURVEY §3.2")
    out = {"impl": "reference", "metric": METRIC, "value": round(mbps, 3), "unit": "MB/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.median(secs), 3),
           "higher_is_better": True, "scaling": "weak" if world == 1 else "strong", "vs_baseline": None,
           "dtype": "u8", "data": "synthetic",
           "config": {"workload": c3_text(1 << 25) if world == 1 else C5_TEXT, "sample": sample},
           "keys_per_s": round(keys_s, 1),
           "cpu_baseline": {"value": round(mbps, 3), "unit": "MB/s", "cores": cores, "kind": kind,
                            "sample": sample},
           "e2e": {"value": round(mbps, 3), "unit": "MB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if args.offload_keys > 0:
        off = bench_ref.offload_throughput(shape, args.offload_keys, max(1, min(args.steps, 3)))
        if off is not None:
            out["offload_host_parallel"] = {"value": round(off[0], 3), "unit": "MB/s", "keys_per_s": round(off[1], 1),
                                            "workers": off[2],
                                            "sample": f"{shape}-shaped job, {args.offload_keys} keys per run"}
    print(json.dumps(out), flush=True)
    return 0


def cpu_baseline(n_keys):
    """Single-core reference compaction on a bounded c3-shaped sample."""
    import bench_ref
    mbps, keys_s, kind, secs = bench_ref.inline_throughput("c3", n_keys, 1, 1, 0)
    return {"value": round(mbps, 4), "unit": "MB/s", "cores": 1, "kind": kind,
            "sample": f"c3-shaped job of 2x{n_keys} entries (16B/128B, 20% deletes), one core: {secs[0]:.1f}s of "
                      f"compaction ({'the pip-installed reference, baseline/_ref' if kind == 'reference' else 'oracle port'})",
            "keys_per_s": round(keys_s, 1)}


# --------------------------------------------------------------------------------------------
# main
# --------------------------------------------------------------------------------------------
def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--keys", type=int, default=1 << 25, help="c3: distinct keys per run (2^25 → 64M entries)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--extras", default="c2,c4,reads,storage,c5", help="other BASELINE configs measured at N=1 ('' = none)")
    ap.add_argument("--c5-gb", type=float, default=256.0, help="c5: global job size (GB of input)")
    ap.add_argument("--cpu-keys", type=int, default=1 << 17,
                    help="reference arm: distinct keys per run of each worker's sample job")
    ap.add_argument("--offload-keys", type=int, default=1 << 15,
                    help="reference arm: keys per run of the host_parallel offload-path sample (0 = skip)")
    ap.add_argument("--cpu-baseline-keys", type=int, default=1 << 20,
                    help="cpu_baseline: distinct keys per run of the single-core sample (~10-30 s)")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def reexec_torchrun(args):
    """`python bench.py --gpus N` without torchrun: one process per GPU."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return reexec_torchrun(args)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
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
        rc = main_c5(args, world, rank, local, backend)
        dist.destroy_process_group()
        return rc
    return main_c3(args, local)


def main_c5(args, world, rank, local, backend):
    """N > 1: BASELINE config 5, strong scaling, max over ranks."""
    import torch
    import torch.distributed as dist
    clocks = ClockSampler(local)
    dist.barrier()
    clocks.start()
    spec, tot = measure_c5(world, rank, local, args.steps, args.warmup, total_gb=args.c5_gb)
    clk = clocks.stop()
    dev = "cuda" if backend == "nccl" else "cpu"
    mx = torch.tensor([tot["ms"], tot["e2e_s"]], dtype=torch.float64, device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = torch.tensor([tot["in_bytes"], tot["n_in"], tot["n_out"], tot["out_bytes"], tot["launches"],
                       tot["e2e_in_bytes"], tot["e2e_h2d"], tot["e2e_d2h"], tot["waves"], tot["staged_bytes"]],
                      dtype=torch.float64, device=dev)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    gathered = [None] * world
    dist.all_gather_object(gathered, {"rank": rank, "ms": round(tot["ms"], 3), "ranges": tot["mine"],
                                      "waves": tot["waves"], "plan_ms": round(tot["plan_ms"], 1),
                                      "wall_s": round(tot["wall_s"], 1), "sm_mhz": clk.get("sm_mhz"),
                                      "reasons": clk.get("reasons")})
    if rank != 0:
        return 0
    ms_max, e2e_s_max = float(mx[0]), float(mx[1])
    in_b, n_in, n_out, out_b, launches, e_in, e_h2d, e_d2h, waves, staged = [float(x) for x in sm.tolist()]
    peaks, peak_kind = load_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    b_alg = in_b + out_b + 2 * 32 * (n_in + n_out) + n_out * 128
    out = {
        "metric": METRIC, "value": round(in_b / (ms_max * 1e-3) / 1e6, 3), "unit": "MB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic (device-synthesised per wave)",
        "config": {"workload": C5_TEXT, "global_input_bytes": int(in_b), "n_in": int(n_in), "n_out": int(n_out),
                   "ranges_P": tot["ranges"], "waves": int(waves), "staged_bytes": int(staged),
                   "parallelism": f"key-range subcompactions, P={tot['ranges']} fixed, {world} GPUs",
                   "step": "one pass of the global job: every rank compacts its ranges (wave time = mean of "
                           "`steps` timed compactions after `warmup`); ms_per_step = max over ranks of the summed "
                           "wave times (CUDA events; synthesis untimed)",
                   "l2": "per-wave inputs (~4 GB) far larger than L2; no flush", "ranks": gathered},
        "keys_per_s": round(n_in / (ms_max * 1e-3), 1),
        "job_roofline": {"alg_bytes": b_alg, "frac": round(b_alg / (ms_max * 1e-3) / 1e9 / (hbm * world), 4),
                         "peak_per_gpu": hbm, "peak_kind": peak_kind},
        "e2e": {"value": round(e_in / e2e_s_max / 1e6, 3) if e2e_s_max else None, "unit": "MB/s",
                "h2d_bytes_per_step": int(e_h2d), "d2h_bytes_per_step": int(e_d2h),
                "timing": "the first 2 waves of every rank run end to end (pinned H2D of the wave's input SSTs + "
                          "job + D2H of its outputs, host clock); value = their owned input bytes summed over "
                          "ranks / the slowest rank's time"},
        "gpu_launches": int(launches), "clocks": clk,
    }
    print(json.dumps(out), flush=True)
    return 0


def main_c3(args, local):
    import torch
    from paper_2004_03054_b200 import _native
    from paper_2004_03054_b200.device import PinnedBuffer
    L = _native.lib(local)
    w = synth_c3(args.keys, seed=0xC3, device_index=local)
    desc, keep = job_desc(w, w.arena.data_ptr())
    st = w.stream

    # correctness spot-check of the job shape
    res = compact_once(L, desc, st)
    assert res.n_in == w.n_in, (res.n_in, w.n_in)
    assert res.n_out == w.n_out_expected, (res.n_out, w.n_out_expected)
    s_out, n_sst = res.out_bytes, res.n_sst
    L.luda_job_release(ctypes.byref(res))
    for _ in range(max(0, args.warmup - 1)):
        L.luda_job_release(ctypes.byref(compact_once(L, desc, st)))

    tm = Timer(L)
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    clocks.start()
    k_acc, t_acc, launches = [0.0] * 8, [0.0] * 8, 0
    tm.start(st)
    for _ in range(args.steps):
        r = compact_once(L, desc, st)
        for i in range(8):
            k_acc[i] += r.k_ms[i]
            t_acc[i] += r.t_ms[i]
        launches += r.launches
        L.luda_job_release(ctypes.byref(r))
    ms_total = tm.stop(st)
    torch.cuda.synchronize()
    t_step = ms_total / args.steps

    # ---- e2e through the public API (run_compactions) with pinned host inputs ----
    e2e = None
    if args.e2e_steps > 0:
        e2e = e2e_public_api(w, args.e2e_steps)
    # ---- the same through the raw C ABI (the floor the API is measured against) ----
    e2e_raw = None
    if args.e2e_steps > 0:
        pin_in, pin_out, pin_out2 = PinnedBuffer(), PinnedBuffer(), PinnedBuffer()
        pin_in.ensure(w.total)
        pin_out.ensure(s_out + 4096)
        pin_out2.ensure(s_out + 4096)
        _native.check(L.luda_stage_out_async(pin_in.ptr, w.arena.data_ptr(), w.total, st))
        _native.check(L.luda_stream_sync(st))
        # Two input arenas: the H2D of step i+1 (in_lower / in_upper streams) runs while step i compacts and
        # step i-1's output streams back (out stream) — PCIe is full duplex.
        arenas = [torch.empty(w.total, dtype=torch.uint8, device="cuda") for _ in range(2)]
        descs = [job_desc(w, ar.data_ptr()) for ar in arenas]
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
            if i > 0:  # job i's copies start when both of job i-1's have landed (same schedule as run_compactions)
                for e in ev_in[(i - 1) % 2]:
                    for sp in (s_lo, s_up):
                        _native.check(L.luda_stream_wait_event(sp.value, e.value))
            _native.check(L.luda_stage_in_async(ar.data_ptr(), pin_in.ptr, split, s_lo.value))
            _native.check(L.luda_stage_in_async(ar.data_ptr() + split, pin_in.ptr + split, w.total - split,
                                                s_up.value))
            _native.check(L.luda_event_record(ev_in[i % 2][0].value, s_lo.value))
            _native.check(L.luda_event_record(ev_in[i % 2][1].value, s_up.value))

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out_bytes, prev = 0, None
        stage(0)
        for i in range(args.e2e_steps):
            if i + 1 < args.e2e_steps:
                stage(i + 1)  # arena (i+1)%2 was last read by job i-1, which has completed
            for e in ev_in[i % 2]:
                _native.check(L.luda_stream_wait_event(st, e.value))
            res = compact_once(L, descs[i % 2][0], st)
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
        e2e_raw = {"value": round(w.s_in / dt / 1e6, 3), "unit": "MB/s", "h2d_bytes_per_step": w.total,
                   "d2h_bytes_per_step": int(out_bytes), "ms_per_step": round(dt * 1e3, 3),
                   "timing": "raw C-ABI calls, same schedule as run_compactions"}
        for p in (pin_in, pin_out, pin_out2):
            p.free()
        del arenas
    clk = clocks.stop()

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

    workloads = {}
    extras = [x for x in args.extras.split(",") if x]
    if "c2" in extras:
        workloads["c2"] = measure_c2(L, st)
    if "c4" in extras:
        workloads["c4_scaled"] = measure_c4(L, st, peak=hbm)
    if "reads" in extras:
        workloads["reads"] = measure_reads(L, desc, st)
    if "storage" in extras:
        workloads["storage"] = measure_storage(L, w, st)
    if "c5" in extras:
        spec, tot = measure_c5(1, 0, local, max(1, args.steps // 5), 1, total_gb=args.c5_gb)
        workloads["c5_1gpu"] = {
            "workload": C5_TEXT + " — 1 GPU (strong-scaling base of the N>1 lines)",
            "value": round(tot["in_bytes"] / (tot["ms"] * 1e-3) / 1e6, 3), "unit": "MB/s",
            "ms_per_step": round(tot["ms"], 3), "global_input_bytes": tot["in_bytes"], "n_in": tot["n_in"],
            "n_out": tot["n_out"], "ranges_P": tot["ranges"], "waves": tot["waves"],
            "plan_ms": round(tot["plan_ms"], 1), "wall_s": round(tot["wall_s"], 1),
            "e2e": {"value": round(tot["e2e_in_bytes"] / tot["e2e_s"] / 1e6, 3) if tot["e2e_s"] else None,
                    "unit": "MB/s", "waves": tot["e2e_waves"]}}
    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline(args.cpu_baseline_keys)
    value = s_in / (t_step * 1e-3) / 1e6
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "MB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": c3_text(args.keys), "keys_per_run": args.keys, "n_in": n_in, "n_out": n_out,
                   "input_bytes": s_in, "output_bytes": int(s_out), "input_ssts": len(w.file_off),
                   "output_ssts": int(n_sst), "block_size": 4096, "sst_size_target": MIB4,
                   "l2": "inputs (%.1f GB) larger than L2; no flush" % (s_in / 1e9), "parallelism": "1 GPU"},
        "keys_per_s": round(n_in / (t_step * 1e-3), 1),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(ach / hbm, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind, "alg_bytes_per_launch": db},
        "job_roofline": {"alg_bytes": b_alg, "achieved": round(b_alg / (t_step * 1e-3) / 1e9, 1), "peak": hbm,
                         "frac": round(b_alg / (t_step * 1e-3) / 1e9 / hbm, 4),
                         "formula": "S_in + S_out + 2(K+8)(N_in+N_out) + V_out"},
        "kernels": kernels,
        "phases_ms": {"parse": round(tms[0], 3), "decode": round(tms[1], 3), "merge": round(tms[2], 3),
                      "plan": round(tms[3], 3), "emit": round(tms[4], 3), "total": round(tms[7], 3)},
        "e2e": e2e,
        "e2e_raw_cabi": e2e_raw,
        "workloads": workloads,
        "gpu_launches": launches,
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
