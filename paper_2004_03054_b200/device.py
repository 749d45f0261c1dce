"""The ``"b200"`` offload device: the reference's plugin protocol on a B200.

Mirrors ``pkg/src/luda/device.py`` (the seam a real-GPU backend was planned
to plug into, SPEC D24): ``make_device(config)`` → an object with
``alloc / free / free_all / stage_in / stage_out / dispatch / stats /
region_in_state / workers / close`` and the ``KernelSpec`` / ``DeviceRegion``
/ ``TransferHandle`` / ``DispatchHandle`` / ``DeviceStatsSnapshot`` types.

* Regions are device allocations (``luda_region_alloc``); the capacity check
  of ``_DeviceBase.alloc`` (device.py:266-281) is kept.
* Named streams ``in_lower`` / ``in_upper`` / ``out`` (device.py:38-40) are
  CUDA streams: FIFO per stream, concurrent across streams. ``stage_in``
  copies the caller's bytes into pinned staging and issues an async H2D copy;
  ``stage_out`` gathers ranges D2H into pinned memory.
* ``dispatch(KernelSpec)`` runs the four reference kernel kinds
  (kernels.py:72-168) as CUDA kernels through ``luda_dispatch``; results come
  back per item in order and the first failing item in dispatch order becomes
  ``CorruptionError(offset)`` / ``DeviceError`` (device.py:392-396, 435-456).
* ``compact(...)`` is the fused job path used by ``run_compaction``.
"""

from __future__ import annotations

import ctypes
import itertools
import threading
import time
from dataclasses import dataclass

from . import _native
from .config import DeviceConfig
from .errors import CapacityError, CorruptionError, DeviceError

STREAM_IN_LOWER = "in_lower"
STREAM_IN_UPPER = "in_upper"
STREAM_OUT = "out"

EMPTY = "empty"
STAGING = "staging"
FILLING = "filling"
READY = "ready"

KERNEL_KINDS = ("unpack", "shared_key", "encode", "filter")
_KIND_ID = {k: i for i, k in enumerate(KERNEL_KINDS)}
_ITEM_COLS = {"unpack": 9, "shared_key": 6, "encode": 10, "filter": 7}
_RESULT_COLS = {"unpack": 4, "shared_key": 1, "encode": 2, "filter": 1}

_region_counter = itertools.count(1)


@dataclass(frozen=True)
class KernelSpec:
    """One dispatch: kernel kind + work-item argument tuples (device.py:112-127)."""

    kind: str
    items: tuple
    reads: tuple = ()
    writes: tuple = ()

    def __post_init__(self):
        if self.kind not in KERNEL_KINDS:
            raise ValueError(f"unknown kernel kind {self.kind!r}")


class DeviceRegion:
    __slots__ = ("region_id", "capacity", "label", "dptr", "_state", "_pending", "_device")

    def __init__(self, region_id, capacity, label, dptr, device):
        self.region_id = region_id
        self.capacity = capacity
        self.label = label
        self.dptr = dptr
        self._state = EMPTY
        self._pending = []
        self._device = device

    @property
    def state(self):
        if self._pending:
            self._pending = [h for h in self._pending if not h.done()]
            if not self._pending and self._state == STAGING:
                self._state = READY
        return self._state

    @state.setter
    def state(self, v):
        self._state = v


class TransferHandle:
    def __init__(self, stream: str, nbytes: int, direction: str, seq: int, event, finish=None):
        self.stream = stream
        self.nbytes = nbytes
        self.direction = direction
        self.seq = seq
        self.t_issue = time.monotonic()
        self.t_start = self.t_issue
        self.t_end = None
        self.error = None
        self._event = event
        self._finish = finish
        self._result = None
        self._done = False
        self._lock = threading.Lock()

    def done(self) -> bool:
        if self._done:
            return True
        if self._event is None:
            return True
        return _native.load().luda_event_query(self._event) == 1

    def wait(self, timeout=None):
        with self._lock:
            if not self._done:
                if self._event is not None:
                    _native.check(_native.load().luda_event_wait(self._event))
                self.t_end = time.monotonic()
                if self._finish is not None:
                    self._result = self._finish()
                self._done = True
        if self.error is not None:
            raise self.error
        return self._result


class DispatchHandle:
    """device.py:167-185: completion is observable from any thread; wait()
    raises the folded error of the first failing item."""

    def __init__(self, kind: str, n_items: int):
        self.kind = kind
        self.n_items = n_items
        self.t_submit = time.monotonic()
        self.t_end = None
        self.results = [None] * n_items
        self.error = None
        self._event = threading.Event()

    def done(self) -> bool:
        return self._event.is_set()

    def wait(self, timeout=None):
        if not self._event.wait(timeout):
            raise DeviceError(f"{self.kind} dispatch timed out")
        if self.error is not None:
            raise self.error
        return self.results


@dataclass
class DeviceStatsSnapshot:
    busy_sec: float
    total_sec: float
    utilization: float
    bytes_in: dict
    bytes_out: dict
    transfer_sec: dict
    dispatches: dict
    items: dict


class _Stats:
    def __init__(self):
        self.lock = threading.Lock()
        self.opened_at = time.monotonic()
        self.busy_total = 0.0
        self.bytes_in, self.bytes_out, self.transfer_sec = {}, {}, {}
        self.dispatches, self.items = {}, {}

    def dispatch(self, kind, n, dt):
        with self.lock:
            self.dispatches[kind] = self.dispatches.get(kind, 0) + 1
            self.items[kind] = self.items.get(kind, 0) + n
            self.busy_total += dt

    def transfer(self, stream, direction, nbytes, dt):
        with self.lock:
            book = self.bytes_in if direction == "in" else self.bytes_out
            book[stream] = book.get(stream, 0) + nbytes
            self.transfer_sec[stream] = self.transfer_sec.get(stream, 0.0) + dt

    def snapshot(self) -> DeviceStatsSnapshot:
        with self.lock:
            total = time.monotonic() - self.opened_at
            return DeviceStatsSnapshot(self.busy_total, total, self.busy_total / total if total > 0 else 0.0,
                                       dict(self.bytes_in), dict(self.bytes_out), dict(self.transfer_sec),
                                       dict(self.dispatches), dict(self.items))


class PinnedBuffer:
    """Grow-only pinned host buffer (cudaHostAlloc)."""

    def __init__(self):
        self.ptr = None
        self.size = 0

    def ensure(self, n: int):
        if n > self.size:
            L = _native.load()
            if self.ptr:
                _native.check(L.luda_host_free(self.ptr))
            p = ctypes.c_void_p()
            _native.check(L.luda_host_alloc(max(n, 1 << 20), ctypes.byref(p)))
            self.ptr, self.size = p.value, max(n, 1 << 20)
        return self.ptr

    def view(self, n: int):
        return (ctypes.c_uint8 * n).from_address(self.ptr)

    def free(self):
        if self.ptr:
            _native.load().luda_host_free(self.ptr)
            self.ptr, self.size = None, 0


class B200Device:
    """CUDA backend of the offload-device protocol."""

    def __init__(self, config: DeviceConfig | None = None):
        self.config = config or DeviceConfig()
        self.ordinal = int(getattr(self.config, "device_ordinal", 0))
        self._L = _native.lib(self.ordinal)
        self._stats = _Stats()
        self._regions: dict[int, DeviceRegion] = {}
        self._alloc_bytes = 0
        self._lock = threading.Lock()
        self._closed = False
        self._streams: dict[str, int] = {}
        self._seq: dict[str, int] = {}
        self._pinned: list = []  # pinned staging kept alive until transfer completion
        self._dispatch_lock = threading.Lock()  # one batched kernel at a time, in submission order
        self._inflight: set = set()  # dispatch handles whose collector thread still runs

    # -- streams --------------------------------------------------------------
    def stream(self, name: str) -> int:
        s = self._streams.get(name)
        if s is None:
            h = ctypes.c_void_p()
            _native.check(self._L.luda_stream_create(ctypes.byref(h)))
            s = self._streams[name] = h.value
        return s

    def _event_on(self, stream_handle):
        e = ctypes.c_void_p()
        _native.check(self._L.luda_event_create(ctypes.byref(e)))
        _native.check(self._L.luda_event_record(e.value, stream_handle))
        return e.value

    # -- regions --------------------------------------------------------------
    def alloc(self, capacity: int, label: str = "") -> DeviceRegion:
        if capacity < 0:
            raise ValueError("negative region capacity")
        with self._lock:
            if self._closed:
                raise DeviceError("device closed")
            if self._alloc_bytes + capacity > self.config.region_capacity:
                raise CapacityError(
                    f"region allocation of {capacity} B exceeds device capacity "
                    f"({self._alloc_bytes} of {self.config.region_capacity} B in use)")
            p = ctypes.c_void_p()
            _native.check(self._L.luda_region_alloc(capacity, ctypes.byref(p)))
            r = DeviceRegion(next(_region_counter), capacity, label, p.value, self)
            self._regions[r.region_id] = r
            self._alloc_bytes += capacity
            return r

    def free(self, region: DeviceRegion):
        with self._lock:
            busy = [h for h in self._inflight if region.region_id in h._rids]
        for h in busy:  # a dispatch still reading / writing the region finishes first
            h._event.wait()
        with self._lock:
            if self._regions.pop(region.region_id, None) is not None:
                self._alloc_bytes -= region.capacity
                for s in self._streams.values():
                    self._L.luda_stream_sync(s)
                _native.check(self._L.luda_region_free(region.dptr))
                region.dptr = None

    def free_all(self):
        for r in list(self._regions.values()):
            self.free(r)

    # -- transfers ------------------------------------------------------------
    def _handle(self, stream, nbytes, direction, event, finish=None):
        seq = self._seq.get(stream, 0)
        self._seq[stream] = seq + 1
        return TransferHandle(stream, nbytes, direction, seq, event, finish)

    def stage_in(self, region: DeviceRegion, data, stream: str, offset: int = 0) -> TransferHandle:
        n = len(data)
        if offset + n > region.capacity:
            raise CapacityError(f"stage_in of {n} B at {offset} exceeds region capacity {region.capacity}")
        if region.state == FILLING:
            raise DeviceError("cannot stage into a region a dispatch is writing")
        region.state = STAGING
        s = self.stream(stream)
        t0 = time.monotonic()
        if n:
            pin = PinnedBuffer()
            pin.ensure(n)
            ctypes.memmove(pin.ptr, (ctypes.c_char * n).from_buffer_copy(bytes(data)) if not isinstance(
                data, (bytes, bytearray)) else bytes(data), n)
            _native.check(self._L.luda_stage_in_async(region.dptr + offset, pin.ptr, n, s))
            self._pinned.append((s, pin))
        ev = self._event_on(s)
        h = self._handle(stream, n, "in", ev)
        region._pending.append(h)
        self._stats.transfer(stream, "in", n, time.monotonic() - t0)
        return h

    def stage_out(self, region: DeviceRegion, ranges, stream: str) -> TransferHandle:
        if region.state in (EMPTY, STAGING):
            raise DeviceError(f"stage_out from region in state {region.state}")
        total = sum(l for _, l in ranges)
        for o, l in ranges:
            if o + l > region.capacity:
                raise CapacityError("stage_out range beyond region capacity")
        s = self.stream(stream)
        pin = PinnedBuffer()
        pin.ensure(total)
        pos = 0
        for o, l in ranges:
            if l:
                _native.check(self._L.luda_stage_out_async(pin.ptr + pos, region.dptr + o, l, s))
            pos += l
        ev = self._event_on(s)

        def finish():
            out = bytes(pin.view(total)) if total else b""
            pin.free()
            return out

        h = self._handle(stream, total, "out", ev, finish)
        self._stats.transfer(stream, "out", total, 0.0)
        return h

    # -- dispatch -------------------------------------------------------------
    def _check_dispatch(self, spec: KernelSpec):
        for rid in spec.reads:
            r = self._regions.get(rid)
            if r is None or r.state != READY:
                raise DeviceError(f"{spec.kind} dispatch reads region {rid} not in ready state")
        for rid in spec.writes:
            r = self._regions.get(rid)
            if r is None or r.state == STAGING:
                raise DeviceError(f"{spec.kind} dispatch writes region {rid} in state "
                                  f"{r.state if r else 'freed'}")
            r.state = FILLING

    def dispatch(self, spec: KernelSpec, on_item=None) -> DispatchHandle:
        if self._closed:
            raise DeviceError("device closed")
        self._check_dispatch(spec)
        h = DispatchHandle(spec.kind, len(spec.items))
        h._rids = set(spec.reads) | set(spec.writes)
        t0 = time.monotonic()

        # Asynchronous like HostParallelDevice.dispatch (device.py:566-607): a
        # collector thread runs the batched kernel, calls on_item(i, result) in
        # item order, then releases the written regions and signals the handle.
        # Dispatches run one at a time per device, in submission order.
        def collect():
            with self._dispatch_lock:
                try:
                    self._run_items(spec, h, on_item)
                except Exception as exc:  # noqa: BLE001 — surfaced at wait()
                    if h.error is None:
                        h.error = exc if isinstance(exc, (DeviceError, CorruptionError)) else \
                            DeviceError(f"dispatch failed: {exc}")
                finally:
                    for rid in spec.writes:
                        r = self._regions.get(rid)
                        if r is not None:
                            r.state = READY
                    h.t_end = time.monotonic()
                    self._stats.dispatch(spec.kind, len(spec.items), h.t_end - t0)
                    with self._lock:
                        self._inflight.discard(h)
                    h._event.set()

        with self._lock:
            self._inflight.add(h)
        th = threading.Thread(target=collect, name=f"luda-collect-{spec.kind}", daemon=True)
        th.start()
        return h

    def _run_items(self, spec: KernelSpec, h: DispatchHandle, on_item):
        n = len(spec.items)
        if n == 0:
            return
        cols = _ITEM_COLS[spec.kind]
        items = (ctypes.c_int64 * (n * cols))()
        for i, it in enumerate(spec.items):
            if len(it) != cols:
                raise DeviceError(f"{spec.kind} item {i} has {len(it)} fields, expected {cols}")
            for j, v in enumerate(it):
                items[i * cols + j] = int(v)
        max_rid = max(self._regions) + 1 if self._regions else 1
        ptrs = (ctypes.c_void_p * max_rid)()
        caps = (ctypes.c_uint64 * max_rid)()
        for rid, r in self._regions.items():
            ptrs[rid] = r.dptr
            caps[rid] = r.capacity
        rcols = _RESULT_COLS[spec.kind]
        res = (ctypes.c_int64 * (n * rcols))()
        fail = ctypes.c_int64(-1)
        # transfers into read regions must land first
        for s in self._streams.values():
            self._L.luda_stream_sync(s)
        st = self._L.luda_dispatch(_KIND_ID[spec.kind], items, n, ptrs, caps, max_rid, res, ctypes.byref(fail),
                                   self.stream("compute"))
        upto = n if fail.value < 0 else fail.value
        for i in range(upto):
            h.results[i] = tuple(int(res[i * rcols + j]) for j in range(rcols))
            if on_item is not None:
                on_item(i, h.results[i])
        if fail.value >= 0 or st != 0:
            msg = self._L.luda_last_error().decode(errors="replace")
            off = self._L.luda_last_error_offset()
            if st == 1:
                h.error = CorruptionError(f"{spec.kind} kernel: {msg}", offset=off if off >= 0 else None)
            else:
                h.error = DeviceError(f"{spec.kind} kernel item failed: {msg}")

    # -- fused job ------------------------------------------------------------
    def compact(self, desc: "_native.JobDesc", stream: str = "compute") -> "_native.JobResult":
        res = _native.JobResult()
        st = self._L.luda_compact(ctypes.byref(desc), ctypes.byref(res), self.stream(stream))
        _native.check(st)
        return res

    def release(self, res):
        self._L.luda_job_release(ctypes.byref(res))

    # -- introspection --------------------------------------------------------
    def stats(self) -> DeviceStatsSnapshot:
        return self._stats.snapshot()

    @property
    def workers(self) -> int:
        return 1

    def region_in_state(self, region: DeviceRegion, state: str) -> bool:
        return region.state == state

    def synchronize(self):
        with self._lock:
            pending = list(self._inflight)
        for h in pending:  # dispatches in flight finish before their regions can go away
            h._event.wait()
        for s in self._streams.values():
            _native.check(self._L.luda_stream_sync(s))
        for _, pin in self._pinned:
            pin.free()
        self._pinned.clear()

    def close(self):
        if self._closed:
            return
        self.synchronize()
        from .compaction import close_runner
        close_runner(self)
        self.free_all()
        for s in self._streams.values():
            self._L.luda_stream_destroy(s)
        self._streams.clear()
        self._closed = True


def make_device(config: DeviceConfig):
    """device.py:622-627 with the ``"b200"`` backend (the only one here: the
    CPU backends stay in the reference; there is no CPU fallback)."""
    if config.backend == "b200":
        return B200Device(config)
    raise ValueError(f"unknown device backend {config.backend!r}")
