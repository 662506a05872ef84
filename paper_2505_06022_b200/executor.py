"""The B200 executor: ``run(plan) -> RunResult`` -- the reference's replaced
seam (pkg/src/clusterq/simulator.py:101-224).

Same inputs and result shape as the reference simulator, but every data-plane
operation is real:

* each plan node is a GPU (``Placement``): in one process, node ``k`` runs on
  device ``k % ndev``; under ``torchrun`` node ``k`` is rank ``k`` (one process
  per GPU, NCCL between ranks -- Celerity's own model, where every rank plans
  the whole program and executes its own commands);
* per (node, buffer) one HBM allocation covering the bounding box of every
  region the node touches;
* Execute -> a kernel launch (see ``lowering``); Push/AwaitPush -> NCCL
  send/recv inside a group, or a DMA copy (same process, NVLink peer copy
  between devices); host-initialised data (version 1, no producer,
  scheduler.py:128-131) is materialised directly on the destination instead
  of being shipped out of node 0;
* final gather -> device-to-host copies of each final piece from its
  lowest-id holder (simulator.py:210-222);
* the trace carries CUDA-event times (seconds, as exact ``Fraction``) so
  ``account_energy`` works unchanged; NVML energy is measured around the run.

Ordering: commands are walked in the reference's Kahn order (lowest ready id
first, simulator.py:108-126).  Local memory hazards are tracked per (node,
buffer) region (RAW/WAR/WAW) and turned into cross-stream event waits, so
independent work overlaps: the rows of an Execute that do not read freshly
received halo cells launch on the compute stream immediately, the dependent
rows go to a high-priority stream after the receive.  Transfers are grouped
between consecutive Executes of the global order (identically on every rank),
and a send and its receive are always posted in the same group.
"""

import ctypes
import heapq
import os
import time
import weakref
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional

import numpy as np

from . import _native as N
from . import fusion, jit
from .errors import EvalError, MapperViolationError, NativeError, ValidationError
from .lowering import bind_task
from .model import AccessMode, NativeKernel, apply_mapper
from .region import Box, Region
from .scheduler import AwaitPushCommand, ExecuteCommand, Plan, PushCommand

# --------------------------------------------------------------- result types


@dataclass(frozen=True)
class LinkModel:
    """Accepted for API compatibility with the reference (simulator.py:35-47);
    the B200 executor measures real transfer times instead of modelling them."""

    latency_s: float = 1e-6
    bandwidth_bytes_per_s: float = 1e9

    def __post_init__(self):
        if self.latency_s < 0:
            raise ValidationError("link latency must be nonnegative")
        if self.bandwidth_bytes_per_s <= 0:
            raise ValidationError("link bandwidth must be positive")

    def transfer_time(self, nbytes: int) -> Fraction:
        return Fraction(self.latency_s) + Fraction(nbytes) / Fraction(self.bandwidth_bytes_per_s)


@dataclass
class TraceEvent:
    kind: str  # "execute" | "push" | "await_push"
    node: int
    command_id: int
    start: Fraction
    duration: Fraction
    bytes: int = 0
    frequency_ghz: Optional[float] = None
    task_id: Optional[int] = None
    task_name: Optional[str] = None
    label: str = ""

    @property
    def finish(self) -> Fraction:
        return self.start + self.duration


@dataclass
class RunResult:
    buffers: dict
    trace: list
    makespan: Fraction
    plan: Plan
    measured: dict = field(default_factory=dict)  # NVML energy, device seconds


def trace_to_chrome(trace) -> list:
    """Chrome trace-viewer events, microseconds (simulator.py:227-246)."""
    lanes = {"execute": 0, "push": 1, "await_push": 2}
    out = []
    for ev in trace:
        args = {"kind": ev.kind, "command": ev.command_id}
        if ev.frequency_ghz is not None:
            args["frequency_ghz"] = ev.frequency_ghz
        if ev.bytes:
            args["bytes"] = ev.bytes
        out.append({"name": ev.label or ev.kind, "ph": "X", "pid": ev.node, "tid": lanes[ev.kind],
                    "ts": float(ev.start * 1_000_000), "dur": float(ev.duration * 1_000_000),
                    "args": args})
    return out


# ------------------------------------------------------------------ placement

@dataclass(frozen=True)
class Placement:
    """node -> (rank, device).  ``world``/``rank`` describe the process group;
    ``devices`` are this process's CUDA devices."""

    world: int
    rank: int
    devices: tuple

    def rank_of(self, node: int, node_count: int) -> int:
        if self.world == 1:
            return 0
        return node * self.world // max(node_count, self.world)

    def device_of(self, node: int, node_count: int) -> int:
        if self.world == 1:
            return self.devices[node % len(self.devices)]
        return self.devices[0]

    def is_local(self, node: int, node_count: int) -> bool:
        return self.rank_of(node, node_count) == self.rank


_dist_state = {"placement": None, "nccl": False}
# page-locked error-flag read-back buffers of closed sessions, by size (reused: never freed)
_FLAG_HOST_CACHE = {}
# counts of collective lowerings this process issued (tests / evidence)
STATS = {"allgather": 0, "bcast": 0, "nccl_groups": 0, "h2d_bytes": 0, "upload_dedup_bytes": 0, "peer_blocks": 0}


def local_placement() -> Placement:
    """Placement of this process: the torchrun rank if NCCL was initialised
    via ``init_distributed``, else all visible GPUs in one process."""
    if _dist_state["placement"] is not None:
        return _dist_state["placement"]
    n = ctypes.c_int32()
    N.call("cq_device_count", ctypes.byref(n))
    if n.value < 1:
        raise ValidationError("no CUDA device visible")
    return Placement(1, 0, tuple(range(n.value)))


def init_distributed(rank: int, world: int, device: int, broadcast_id=None) -> Placement:
    """Create this rank's NCCL communicator (one rank per GPU).

    ``broadcast_id(bytes_or_None) -> bytes`` distributes rank 0's NCCL unique
    id; by default it uses ``torch.distributed`` (already initialised, any
    backend) purely as plumbing."""
    if broadcast_id is None:
        def broadcast_id(blob):
            import torch.distributed as dist
            box = [blob]
            dist.broadcast_object_list(box, src=0)
            return box[0]
    uid = None
    if rank == 0:
        buf = ctypes.create_string_buffer(128)
        N.call("cq_nccl_unique_id", buf)
        uid = buf.raw
    uid = broadcast_id(uid)
    N.call("cq_init_device", device)
    if world > 1:
        N.call("cq_nccl_init", device, world, rank, uid)
        _dist_state["nccl"] = True
    pl = Placement(world, rank, (device,))
    _dist_state["placement"] = pl
    return pl


def shutdown_distributed():
    if _dist_state["nccl"]:
        N.call("cq_nccl_destroy")
    _dist_state.update(placement=None, nccl=False)


# ---------------------------------------------------------------- host memory

# Page-locked spans of host arrays: (start, end) -> weakref.finalize that
# unregisters the span when the array owning the memory is garbage-collected
# (so registrations live exactly as long as the arrays, and repeated runs
# over the same inputs register them once), or a strong reference for memory
# no ndarray owns.
_pinned = {}
_temp_spans = set()
_PAGE = 4096
# Only arrays this large are page-locked: glibc serves them from their own
# mmap'd pages, so a registration never shares a page with another array.
PIN_MIN_BYTES = 64 << 20


def _byte_span(arr, box):
    if box is None:
        return arr.ctypes.data, arr.ctypes.data + arr.nbytes
    lo = sum(m * s for m, s in zip(box.mins, arr.strides))
    hi = sum((m - 1) * s for m, s in zip(box.maxs, arr.strides)) + arr.itemsize
    return arr.ctypes.data + lo, arr.ctypes.data + hi


def _pin_state(start, end):
    """"pinned" (inside one registration), "partial" (overlaps one -- a DMA
    over it would be invalid) or "free" (pageable, no registration)."""
    for s, e in list(_pinned) + list(_temp_spans):
        if s <= start and end <= e:
            return "pinned"
        if s < end and start < e:
            return "partial"
    return "free"


def _free_scratch(items):
    """Free (device, pointer | _View) temporaries and empty the list."""
    for dev, item in items:
        if isinstance(item, _View):
            item.free()
        else:
            N.call("cq_free", dev, ctypes.c_void_p(item))
    items.clear()


def _raise_flag(code, point):
    """The reference's exception for a device error-flag code."""
    if code == N.CQ_ERR_EVAL:
        raise EvalError(f"integer division by zero at id {point}")
    if code == N.CQ_ERR_MAPPER:
        raise MapperViolationError(f"read at id {point} outside the mapped region")
    if code == N.CQ_ERR_P2P:
        raise NativeError(f"a neighbour's halo signal did not arrive (wanted pass {point[0]}, saw {point[1]})")


def _memory_owner(arr):
    """The ndarray that owns ``arr``'s memory (walking view bases), or None."""
    o = arr
    while isinstance(o, np.ndarray) and o.base is not None:
        o = o.base
    return o if isinstance(o, np.ndarray) and o.base is None else None


def _unregister_span(span):
    if _pinned.pop(span, None) is not None:
        try:
            N.call("cq_host_unregister", ctypes.c_void_p(span[0]))
        except Exception:  # noqa: BLE001  (interpreter shutdown / library gone)
            pass


def _pin_span(arr: np.ndarray, box=None, keep=True):
    """Page-lock the bytes of a large ``arr`` spanning ``box`` (whole array if
    None); a rank of a weak-scaled run pins only its own rows of a big host
    array.  keep=True: the registration lasts until the array owning the
    memory is garbage-collected (or ``release_pinned``).  Returns the span
    when registered temporarily (keep=False)."""
    if arr.nbytes < PIN_MIN_BYTES:
        return None
    a, b = _byte_span(arr, box)
    start = a // _PAGE * _PAGE
    end = -(-b // _PAGE) * _PAGE
    if _pin_state(start, end) != "free":
        return None
    N.call("cq_host_register", ctypes.c_void_p(start), end - start)
    if keep:
        owner = _memory_owner(arr)
        if owner is not None:
            fin = weakref.finalize(owner, _unregister_span, (start, end))
            fin.atexit = False
            _pinned[(start, end)] = fin
        else:
            _pinned[(start, end)] = arr
        return None
    _temp_spans.add((start, end))
    return (start, end)


def _needs_bounce(arr, box):
    """True when a DMA over ``box`` of ``arr`` would straddle a registration
    edge; such copies go through a temporary pageable array instead."""
    return _pin_state(*_byte_span(arr, box)) == "partial"


def _unpin_temp(span):
    N.call("cq_host_unregister", ctypes.c_void_p(span[0]))
    _temp_spans.discard(span)


def _pin(arr: np.ndarray):
    _pin_span(arr, None, keep=True)


def release_pinned():
    """Unregister every kept registration now (they otherwise end with
    their arrays)."""
    for span, holder in list(_pinned.items()):
        if isinstance(holder, weakref.finalize):
            holder.detach()
        _pinned.pop(span, None)
        N.call("cq_host_unregister", ctypes.c_void_p(span[0]))


def pinned_empty(shape, dtype, box=None) -> np.ndarray:
    """A host array page-locked over ``box`` (whole array if None) for the
    inputs / outputs of repeated runs."""
    arr = np.empty(shape, dtype=dtype)
    _pin_span(arr, box, keep=True)
    return arr


# ------------------------------------------------------------ region helpers

def _pad(box: Box):
    """3-D padded bounds (leading unit axes)."""
    pad = 3 - box.dims
    return (0,) * pad + box.mins, (1,) * pad + box.maxs


def _cbox(box: Box) -> N.CqBox:
    return N.box3(box.mins, box.maxs)


def _bbox_union(boxes):
    boxes = [b for b in boxes if b is not None]
    if not boxes:
        return None
    lo = tuple(min(b.mins[k] for b in boxes) for k in range(boxes[0].dims))
    hi = tuple(max(b.maxs[k] for b in boxes) for k in range(boxes[0].dims))
    return Box(lo, hi)


class _View:
    """One (node, buffer) HBM allocation."""

    __slots__ = ("node", "device", "buffer", "box", "ptr", "c", "itemsize", "nbytes")

    def __init__(self, node, device, buffer, box, itemsize):
        self.node, self.device, self.buffer, self.box = node, device, buffer, box
        self.itemsize = itemsize
        lo, hi = _pad(box)
        shape = [h - l for l, h in zip(lo, hi)]
        self.nbytes = shape[0] * shape[1] * shape[2] * itemsize
        p = ctypes.c_void_p()
        N.call("cq_malloc", device, max(self.nbytes, 16), ctypes.byref(p))
        self.ptr = p.value
        v = N.CqView()
        v.ptr = self.ptr
        v.alloc.lo[:] = lo
        v.alloc.hi[:] = hi
        v.stride[:] = [shape[1] * shape[2], shape[2], 1]
        self.c = v

    def free(self):
        if self.ptr:
            N.call("cq_free", self.device, ctypes.c_void_p(self.ptr))
            self.ptr = None

    def addr(self, point):
        """Device address of global cell ``point`` (unpadded)."""
        lo, _ = _pad(self.box)
        p = (0,) * (3 - len(point)) + tuple(point)
        off = sum((a - b) * s for a, b, s in zip(p, lo, self.c.stride))
        return self.ptr + off * self.itemsize


class _PeerView:
    """A peer rank's allocation opened through CUDA IPC (device pointer valid
    in this process): the ``c`` view of a copy destination, never freed here."""

    __slots__ = ("ptr", "c")

    def __init__(self, ptr, box):
        lo, hi = _pad(box)
        shape = [h - l for l, h in zip(lo, hi)]
        self.ptr = ptr
        v = N.CqView()
        v.ptr = ptr
        v.alloc.lo[:] = lo
        v.alloc.hi[:] = hi
        v.stride[:] = [shape[1] * shape[2], shape[2], 1]
        self.c = v


class _PeerHalo:
    """The halo rows of a temporally blocked chain written straight into the
    neighbouring ranks' allocations over NVLink, instead of one NCCL exchange
    per block.  The NCCL exchange's kernel needs SM slots the running pass
    holds, so it finished only as the pass drained and the edge launches ran
    after it (~30 us per pass at N=2, ~60 at N=4; profiles/r02/
    halo_timeline_n2.log).  Here every block is one launch over the whole
    slab (cq_wave5_fused_ex with cq_mirror_t / cq_peer_sync_t): the pieces
    next to a neighbour first wait, in the kernel, until that neighbour has
    finished the previous block (its rows for this block are in place, and it
    no longer reads the rows this block sends it), and at their end store
    their rows next to the neighbour, of both output fields, into the
    neighbour's output allocation (CUDA IPC pointers, NVLink), raise its |X|
    bound, and the last of them bumps and publishes this rank's pass counter.
    Interior pieces never wait.  The chain's first block reads its halo
    through the plan's NCCL exchange as before; a trailing cq_p2p_wait orders
    the neighbours' last rows before anything else touches the halo rows."""

    TIMEOUT_NS = 30_000_000_000   # a wait that long is a bug (or a stalled rank): the device flag reports it

    def __init__(self, sess, ch):
        self.s = sess
        me = self.me = sess.pl.rank
        self.lo, self.hi = ch.rows[me]
        self.top = next((n for n, (_l, h) in ch.rows.items() if h == self.lo), None)
        self.bot = next((n for n, (l, _h) in ch.rows.items() if l == self.hi), None)
        self.dev = sess.dev(me)
        self.bufs = (ch.a, ch.b)
        self.mine = {buf: (sess.views[(me, buf)], sess.alt[(me, buf)]) for buf in self.bufs}
        # signal words: [0] written by the top neighbour, [1] by the bottom one, [2] this rank's pass
        # count, [3] the pass's finished edge blocks
        p = ctypes.c_void_p()
        N.call("cq_malloc", self.dev, 64, ctypes.byref(p))
        self.sig = p.value
        zero = np.zeros(8, np.uint64)
        N.call("cq_copy_h2d", self.dev, N.STREAM_COMM, p, ctypes.c_void_p(zero.ctypes.data), 64)
        N.call("cq_stream_synchronize", self.dev, N.STREAM_COMM)
        # the per-block |X| bounds (float32 chains): edge blocks raise the
        # neighbours' too, so every piece keeps the FMA form
        self.amax = sess._amax.get((sess.chains.index(ch), me))
        ptrs = [v.ptr for buf in self.bufs for v in self.mine[buf]] + [self.sig]
        if self.amax is not None:
            ptrs.append(self.amax)
        self.peer, self.opened = {}, []
        # every step below is collective: a rank that cannot export or open
        # IPC handles says so, and then every rank falls back together
        try:
            blob = b"\x01" + b"".join(self._handle(x) for x in ptrs)
        except NativeError:
            blob = b"\x00" * (1 + 64 * len(ptrs))
        table = sess.allgather_bytes(blob)
        ok = all(t[0] == 1 for t in table)
        if ok:
            try:
                for nbr in (self.top, self.bot):
                    if nbr is None:
                        continue
                    theirs = [self._open(table[nbr][1 + 64 * i:1 + 64 * (i + 1)]) for i in range(len(ptrs))]
                    entry = {}
                    for k, buf in enumerate(self.bufs):
                        box = sess._alloc_box[(nbr, buf)]
                        entry[buf] = (_PeerView(theirs[2 * k], box), _PeerView(theirs[2 * k + 1], box))
                    entry["sig"] = theirs[4]
                    entry["amax"] = theirs[5] if self.amax is not None else None
                    self.peer[nbr] = entry
            except NativeError:
                ok = False
            ok = all(t == b"\x01" for t in sess.allgather_bytes(b"\x01" if ok else b"\x00"))
        self.ok = ok
        if not ok:
            self.close()

    def _handle(self, ptr):
        h = (ctypes.c_ubyte * 64)()
        N.call("cq_ipc_handle", ctypes.c_void_p(ptr), h)
        return bytes(h)

    def _open(self, handle):
        p = ctypes.c_void_p()
        N.call("cq_ipc_open", self.dev, (ctypes.c_ubyte * 64).from_buffer_copy(handle), ctypes.byref(p))
        self.opened.append(p.value)
        return p.value

    def close(self):
        for p in self.opened:
            try:
                N.call("cq_ipc_close", self.dev, ctypes.c_void_p(p))
            except NativeError:
                pass
        self.opened = []
        if self.sig:
            N.call("cq_free", self.dev, ctypes.c_void_p(self.sig))
            self.sig = None

    def _halo_rows(self, kl, W, views):
        """(view, halo-row region, write) of the rows the neighbours write."""
        boxes = []
        if self.top is not None:
            boxes.append(Box((self.lo - kl, 0), (self.lo, W)))
        if self.bot is not None:
            boxes.append(Box((self.hi, 0), (self.hi + kl, W)))
        if not boxes:
            return []
        reg = Region(2, boxes)
        return [(v, reg, True) for v in views]

    def wait(self, kl, W, views):
        """Stream waits until both neighbours have finished as many blocks as
        this rank; registered as a write of the halo rows the neighbours
        write, so later local users of those rows order after it."""
        s, dev, lane = self.s, self.dev, self.s.lane(self.me)
        slot_t = ctypes.c_void_p(self.sig) if self.top is not None else None
        slot_b = ctypes.c_void_p(self.sig + 8) if self.bot is not None else None

        def go():
            N.call("cq_p2p_wait", dev, lane, slot_t, slot_b, ctypes.c_void_p(self.sig + 16), self.TIMEOUT_NS)
        return s.issue(dev, lane, self._halo_rows(kl, W, views), go)

    def mirrors(self, depth, outs):
        """cq_mirror_t array for the pass writing ``outs`` (X(t+KL), X(t+KL-1)):
        the ``depth`` rows next to each neighbour also go to that neighbour's
        output allocations (the same slot on every rank: lock-step swaps)."""
        arr = (N.CqMirror * 2)()
        n = 0
        for nbr, (r0, r1) in ((self.top, (self.lo, self.lo + depth)), (self.bot, (self.hi - depth, self.hi))):
            if nbr is None:
                continue
            dst = [self.peer[nbr][buf][0 if out is self.mine[buf][0] else 1] for buf, out in zip(self.bufs, outs)]
            m = arr[n]
            m.last, m.prev = dst[0].ptr, dst[1].ptr
            m.row0, m.col0, m.stride = dst[0].c.alloc.lo[1], dst[0].c.alloc.lo[2], dst[0].c.stride[1]
            m.row_lo, m.row_hi = r0, r1
            n += 1
        return arr, n

    def sync(self, bi):
        """cq_peer_sync_t of this rank's passes: the edge blocks wait for the
        neighbours' counters (words [0] / [1] here) to reach this rank's count
        (word [2]); the last edge block bumps it and stores it into the
        neighbours' words ([1] of the top one, [0] of the bottom one); word
        [3] counts the pass's finished edge blocks."""
        sy = N.CqPeerSync()
        if self.top is not None:
            sy.slot[0] = self.sig
            sy.peer_slot[0] = self.peer[self.top]["sig"] + 8
        if self.bot is not None:
            sy.slot[1] = self.sig + 8
            sy.peer_slot[1] = self.peer[self.bot]["sig"]
        sy.count, sy.done = self.sig + 16, self.sig + 24
        for k, nbr in enumerate((self.top, self.bot)):
            if nbr is not None and self.peer[nbr]["amax"] is not None:
                sy.peer_amax[k] = self.peer[nbr]["amax"] + 4 * (bi + 1)   # their bound after block bi
        sy.timeout_ns = self.TIMEOUT_NS
        return sy


# ------------------------------------------------------------- hazard tracker

class _Hazards:
    """Per physical allocation list of recent accesses -> events to wait on.

    An access is (key, region, write?) with key = the allocation (a view's
    id, so the alternate arrays of a fused wave chain are tracked apart even
    as they swap roles).  A new op on stream S waits for every conflicting
    access (RAW, WAR, WAW) issued on another stream; same-stream order is
    implicit.  Entries covered by a newer write, or by a newer access on the
    same stream, can never be the binding constraint again and are dropped."""

    def __init__(self):
        self.log = {}

    def waits(self, accesses, skey):
        out = {}
        for key, region, write in accesses:
            for r, w, sk, ev in self.log.get(key, ()):
                if sk == skey or not (write or w):
                    continue
                if region.overlaps(r):
                    out[ev] = sk
        return out

    def record(self, accesses, skey, event):
        for key, region, write in accesses:
            kept = []
            for entry in self.log.get(key, ()):
                r, w, sk, ev = entry
                if (write or sk == skey) and region.contains_region(r):
                    continue
                kept.append(entry)
            kept.append((region, write, skey, event))
            self.log[key] = kept


# ------------------------------------------------------------------ the run

def kahn_order(plan: Plan) -> list:
    """Lowest-ready-id-first topological order (simulator.py:108-126);
    raises ValidationError on a cycle (simulator.py:204-206)."""
    cached = getattr(plan, "_cq_order", None)
    if cached is not None and cached[0] == len(plan.commands):
        return cached[1]
    indeg = {c.id: len(c.deps) for c in plan.commands}
    users = {c.id: [] for c in plan.commands}
    for c in plan.commands:
        for d in c.deps:
            users[d].append(c.id)
    heap = [cid for cid, d in indeg.items() if d == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        cid = heapq.heappop(heap)
        order.append(cid)
        for u in users[cid]:
            indeg[u] -= 1
            if indeg[u] == 0:
                heapq.heappush(heap, u)
    if len(order) != len(plan.commands):
        stuck = sorted(cid for cid, d in indeg.items() if d > 0)
        raise ValidationError(f"command graph has a cycle involving ids {stuck}")
    plan._cq_order = (len(plan.commands), order)
    return order


class Session:
    """A plan bound to this process's GPUs: allocations persist across
    ``execute`` calls, so a program can be re-run on device-resident data.

    ``run()`` is one upload + execute + gather; benchmarks use the pieces."""

    def __init__(self, plan: Plan, placement: Optional[Placement] = None, trace: bool = True,
                 copy_streams=None, peer_halo: bool = True):
        placement = placement or local_placement()
        self.plan = plan
        # fused wave blocks store their halo rows straight into the
        # neighbouring ranks' memory (_PeerHalo) when allowed; see
        # _peer_halo_for for the environment override
        self.peer_halo = peer_halo
        # streams of the host uploads / read-backs (default: the comm stream);
        # run_batch gives its two sessions their own, so one session's
        # read-back, the other's upload and the kernels overlap
        self.h2d_stream, self.d2h_stream = copy_streams or (N.STREAM_COMM, N.STREAM_COMM)
        self.pl = placement
        self.want_trace = trace
        self.buffers = plan.graph.buffers
        self.by_id = {c.id: c for c in plan.commands}
        self.nodes = plan.node_count
        self.local_nodes = [n for n in range(self.nodes) if placement.is_local(n, self.nodes)]
        self.devices = sorted({placement.device_of(n, self.nodes) for n in self.local_nodes})
        self.views = {}
        self.scratch = []         # this run's temporaries (freed by recycle)
        self._graph_scratch = []  # temporaries a captured graph uses (freed with it)
        self._slots = []          # session-lifetime device words (fused-chain bounds)
        self.events = []
        self.free_events = {}
        self.haz = _Hazards()
        self.bindings = {}
        self.trace_marks = []   # per command: timing events for the trace
        self.launch_log = []    # (binding kind, cells, device, start, stop) per kernel launch
        self.capturing = False
        self.graph = None
        self.graphs = []        # one graph, or two alternating ones (odd fused chains)
        self._graph_logs = []
        self._phase = 0         # which of two graphs launches next
        self.graph_log = []     # launch_log of a timed capture: its events re-record per replay
        self.graph_events = []
        self.host_init = {}
        self._overridden = set()
        self._flag_host = None   # page-locked copies of the devices' error flags (run_batch)
        self._sched = None
        self._raw = None        # the plan's schedule before fusion (schedule())
        self._lanes = None      # node -> compute stream (lane())
        self._exec_of = None    # (task id, node) -> ExecuteCommand (exec_fused)
        self._jcols = None      # N-body j columns (cq_nbody_jcols)
        self._peer = {}         # chain index -> _PeerHalo or None (peer-memory halo rows)
        self._halo_marks = []   # trace marks of a fused block's halo transfers
        self.t0 = None
        self._t0 = {}
        self.uploading = True
        self.bounce = []        # temporaries of bounced host copies (kept until sync)
        kahn_order(plan)  # validates acyclicity before touching devices
        for d in self.devices:
            N.call("cq_init_device", d)
        # several GPUs in one process: box copies between them go peer to
        # peer over NVLink (they stay correct, staged, without it)
        for d in self.devices:
            for e in self.devices:
                if d != e:
                    ok = ctypes.c_int32()
                    N.call("cq_enable_peer", d, e, ctypes.byref(ok))
        self.alt = {}
        self.chains = fusion.find_chains(plan, self._raw_schedule())
        self.allocate()
        self.pin_inputs()

    def pin_inputs(self):
        """Page-lock, once per process, the span of each host input array
        that this process uploads (node 0's copy and version-1 destinations)."""
        need = {}
        for (node, buf), view in self.views.items():
            if node == 0 and self.buffers[buf].init.kind in ("array", "values"):
                need.setdefault(buf, []).append(self.seed_box.get((node, buf)) or view.box)
        for c in self.plan.commands:
            if isinstance(c, PushCommand) and not c.deps and self.local(c.dst) \
                    and self.buffers[c.buffer].init.kind in ("array", "values"):
                need.setdefault(c.buffer, []).append(c.region.bounding_box())
        for buf, boxes in need.items():
            _pin_span(self.host_array(buf), _bbox_union(boxes), keep=True)

    # ---- small helpers -------------------------------------------------
    def dev(self, node):
        return self.pl.device_of(node, self.nodes)

    def local(self, node):
        return self.pl.is_local(node, self.nodes)

    def rank(self, node):
        return self.pl.rank_of(node, self.nodes)

    def event(self, device, timing=False):
        pool = self.free_events.setdefault((device, timing), [])
        if pool:
            ev = pool.pop()
        else:
            h = ctypes.c_uint64()
            N.call("cq_event_create", device, 1 if timing else 0, ctypes.byref(h))
            ev = h.value
        self.events.append((device, timing, ev))
        return ev

    def issue(self, device, stream, accesses, fn):
        """Run ``fn`` on (device, stream) after the hazards it depends on.
        Returns (start, stop) events; ``start`` is None unless tracing."""
        skey = (device, stream)
        accesses = self._keyed(accesses)
        for ev, _sk in self.haz.waits(accesses, skey).items():
            N.call("cq_stream_wait_event", device, stream, ctypes.c_uint64(ev))
        start = tstop = None
        if self.want_trace:
            start = self.event(device, timing=True)
            N.call("cq_event_record_timed", ctypes.c_uint64(start), device, stream)
        fn()
        if self.want_trace and self.capturing:
            # inside a capture the hazard event only becomes a graph edge;
            # the timestamp needs its own event-record node
            tstop = self.event(device, timing=True)
            N.call("cq_event_record_timed", ctypes.c_uint64(tstop), device, stream)
        stop = self.event(device, timing=self.want_trace and not self.capturing)
        N.call("cq_event_record", ctypes.c_uint64(stop), device, stream)
        self.haz.record(accesses, skey, stop)
        return start, tstop or stop

    def _keyed(self, accesses):
        """(node, buffer, region, write) -> (allocation key, region, write) for
        the node's current view; (view, region, write) names a view directly."""
        out = []
        for acc in accesses:
            if len(acc) == 3:
                view, region, write = acc
                out.append((id(view), region, write))
            else:
                node, buf, region, write = acc
                v = self.views.get((node, buf))
                out.append((id(v) if v is not None else (node, buf), region, write))
        return out

    # ---- allocation ----------------------------------------------------
    def allocate(self):
        touch = {}
        for c in self.plan.commands:
            if isinstance(c, ExecuteCommand):
                for _a, buf, reg in c.reads:
                    touch.setdefault((c.node, buf), []).append(reg.bounding_box())
                for _a, buf, reg, _v in c.writes:
                    touch.setdefault((c.node, buf), []).append(reg.bounding_box())
            elif isinstance(c, PushCommand):
                bb = c.region.bounding_box()
                if c.deps:
                    # host-initialised pushes are uploaded at the destination,
                    # so their source never holds the region on a device
                    touch.setdefault((c.src, c.buffer), []).append(bb)
                touch.setdefault((c.dst, c.buffer), []).append(bb)
        for name, entries in self.plan.final_locations.items():
            init = self.buffers[name].init.is_initialized
            for reg, version, holders in entries:
                if init and version == 1:
                    continue  # gathered straight from the host array
                for h in holders:
                    touch.setdefault((h, name), []).append(reg.bounding_box())
        # what node 0 uploads: everything it touches in the plan itself (the
        # deeper fused halo rows are filled by the first exchange)
        self.seed_box = {k: _bbox_union(v) for k, v in touch.items()}
        fused = set()
        for ch in self.chains:
            # fused blocks read a KL-deep halo and write out of place
            for node, (lo, hi) in ch.rows.items():
                for buf in (ch.a, ch.b):
                    touch.setdefault((node, buf), []).append(
                        Box((max(lo - ch.depth, 0), 0), (min(hi + ch.depth, ch.H), ch.W)))
                    fused.add((node, buf))
        self._alloc_box = {k: _bbox_union(v) for k, v in touch.items()}
        for (node, buf), boxes in sorted(touch.items()):
            if not self.local(node):
                continue
            bb = _bbox_union(boxes)
            if bb is None:
                continue
            b = self.buffers[buf]
            self.views[(node, buf)] = _View(node, self.dev(node), buf, bb, b.itemsize)
            if (node, buf) in fused:
                self.alt[(node, buf)] = _View(node, self.dev(node), buf, bb, b.itemsize)
        # per float32 chain and local node: one device float per block
        # boundary, max |X| over the node's rows after that block (written by
        # the block's launches, read by the next: cq_wave5_fused_bounded).
        # Zeroed once; later runs only raise them, which keeps them bounds.
        self._amax = {}
        for ci, ch in enumerate(self.chains):
            if self.buffers[ch.a].element_kind != "float32":
                continue
            for node in sorted(ch.rows):
                if not self.local(node):
                    continue
                dev, n = self.dev(node), len(ch.blocks) + 1
                p = ctypes.c_void_p()
                N.call("cq_malloc", dev, 4 * n, ctypes.byref(p))
                zero = np.zeros(n, np.float32)
                N.call("cq_copy_h2d", dev, N.STREAM_COMPUTE, p, ctypes.c_void_p(zero.ctypes.data), 4 * n)
                N.call("cq_stream_synchronize", dev, N.STREAM_COMPUTE)
                self._slots.append((dev, p.value))
                self._amax[(ci, node)] = p.value

    # ---- host-initialised data -----------------------------------------
    def host_array(self, buf):
        """Host copy of a buffer's initial contents (array inits by reference)."""
        arr = self.host_init.get(buf)
        if arr is None:
            b = self.buffers[buf]
            arr = np.ascontiguousarray(b.init.materialize(b.extent, b.element_kind))
            self.host_init[buf] = arr
        return arr

    def materialize(self, node, buf, region, stream):
        """Write host-initialised contents of ``region`` into node's view."""
        b = self.buffers[buf]
        view = self.views[(node, buf)]
        dev = view.device
        init = b.init
        kind = N.KIND_CODE[b.element_kind]
        ext = _cbox(b.extent)

        def go():
            for box in region.boxes:
                cb = _cbox(box)
                if init.kind in ("array", "values"):
                    arr = self.host_array(buf)
                    if _needs_bounce(arr, box):
                        sl = tuple(slice(lo, hi) for lo, hi in zip(box.mins, box.maxs))
                        tmp = np.array(arr[sl], copy=True)  # never a view of the pinned array
                        self.bounce.append(tmp)
                        N.call("cq_copy_box_h2d", dev, stream, b.itemsize, ctypes.byref(view.c),
                               ctypes.c_void_p(tmp.ctypes.data), ctypes.byref(cb), ctypes.byref(cb))
                        continue
                    N.call("cq_copy_box_h2d", dev, stream, b.itemsize, ctypes.byref(view.c),
                           ctypes.c_void_p(arr.ctypes.data), ctypes.byref(ext), ctypes.byref(cb))
                    STATS["h2d_bytes"] += box.volume() * b.itemsize
                else:
                    mode = {"iota": 1, "constant": 2}.get(init.kind, 0)
                    val = float(init.value) if init.kind == "constant" else 0.0
                    ival = int(init.value) if (init.kind == "constant" and b.element_kind == "int64") else 0
                    N.call("cq_fill", dev, stream, kind, ctypes.byref(view.c), ctypes.byref(cb),
                           ctypes.byref(ext), mode, ctypes.c_double(val), ival)
        return self.issue(dev, stream, [(node, buf, region, True)], go)

    def seed_node0(self):
        """Node 0 holds version 1 of every initialised buffer; materialise it
        over node 0's allocation (only what node 0 itself touches)."""
        if not self.local(0):
            return
        # buffers initialised from the same host array (e.g. a wave's u0 and
        # up0 = u0) cross PCIe once: the others copy it device to device
        # (before any kernel, so the first copy still holds version 1)
        first = {}
        for (node, buf), view in self.views.items():
            if node != 0 or not self.buffers[buf].init.is_initialized:
                continue
            box = self.seed_box.get((node, buf)) or view.box
            region = Region.from_box(box)
            src = self._uploaded_within(first, 0, buf, box)
            if src is not None:
                self.device_copy(0, src, buf, region, self.h2d_stream)
                continue
            self.materialize(0, buf, region, self.h2d_stream)
            self._note_upload(first, 0, buf, box)

    def _host_ident(self, buf):
        """Identity of the host bytes an array-initialised buffer uploads
        from (None for other inits)."""
        b = self.buffers[buf]
        if b.init.kind != "array":
            return None
        arr = self.host_array(buf)
        return (arr.__array_interface__["data"][0], arr.dtype.str, arr.shape, arr.strides)

    def _uploaded_within(self, first, node, buf, box):
        """A buffer whose node allocation (same device) already received the
        same host bytes over a box containing ``box`` -- e.g. u's slab plus
        its halo row when up (same host array, no halo) follows -- or None."""
        ident = self._host_ident(buf)
        if ident is None:
            return None
        dev = self.views[(node, buf)].device
        for sbox, sbuf in first.get((node, ident), ()):
            if sbox.contains_box(box) and self.views[(node, sbuf)].device == dev:
                return sbuf
        return None

    def _note_upload(self, first, node, buf, box):
        ident = self._host_ident(buf)
        if ident is not None:
            first.setdefault((node, ident), []).append((box, buf))

    def device_copy(self, node, src_buf, dst_buf, region, stream):
        """``region`` of node's ``src_buf`` allocation into its ``dst_buf`` one."""
        src, dst = self.views[(node, src_buf)], self.views[(node, dst_buf)]
        eb = self.buffers[dst_buf].itemsize

        def go():
            for box in region.boxes:
                N.call("cq_copy_box", dst.device, stream, eb, ctypes.byref(dst.c), dst.device, ctypes.byref(src.c),
                       src.device, ctypes.byref(_cbox(box)))
                STATS["upload_dedup_bytes"] += box.volume() * eb
        return self.issue(dst.device, stream, [(node, src_buf, region, False), (node, dst_buf, region, True)], go)

    # ---- transfers -------------------------------------------------------
    def flush_group(self, group):
        """Issue one group of transfers (all ranks cut groups identically)."""
        if not group:
            return
        nccl_ops = []
        first = {}   # (node, host bytes) -> [(box, buffer)] materialised there in this group
        for push in group:
            src_l, dst_l = self.local(push.src), self.local(push.dst)
            if not push.deps:
                # host-initialised data: the destination materialises it; the
                # same host bytes for a second buffer are a device copy
                if dst_l and self.uploading:
                    box = push.region.bounding_box()
                    single = len(push.region.boxes) == 1
                    src = self._uploaded_within(first, push.dst, push.buffer, box) if single else None
                    if src is not None:
                        t = self.device_copy(push.dst, src, push.buffer, push.region, self.h2d_stream)
                    else:
                        t = self.materialize(push.dst, push.buffer, push.region, self.h2d_stream)
                        if single:
                            self._note_upload(first, push.dst, push.buffer, box)
                    self.mark_transfer(push, push.dst, t)
                continue
            if src_l and dst_l:
                self.local_copy(push)
            elif src_l or dst_l:
                nccl_ops.append(push)
        if nccl_ops:
            # the 'all' exchange is recognised on the whole group (identical
            # on every rank), then this rank's part of it posted
            dev_pushes = [p for p in group if p.deps]
            layout = self._allgather_layout(dev_pushes)
            bcast = self._bcast_layout(dev_pushes) if layout is None else None
            if layout is not None:
                self.allgather(nccl_ops, *layout)
            elif bcast is not None:
                self.bcast(nccl_ops, *bcast)
            else:
                self.nccl_group(nccl_ops)

    def local_copy(self, push):
        src = self.views[(push.src, push.buffer)]
        dst = self.views[(push.dst, push.buffer)]
        dev = dst.device
        eb = self.buffers[push.buffer].itemsize
        acc = [(push.src, push.buffer, push.region, False), (push.dst, push.buffer, push.region, True)]

        def go():
            for box in push.region.boxes:
                cb = _cbox(box)
                N.call("cq_copy_box", dev, N.STREAM_COMM, eb, ctypes.byref(dst.c), dst.device,
                       ctypes.byref(src.c), src.device, ctypes.byref(cb))
        self.mark_transfer(push, push.dst, self.issue(dev, N.STREAM_COMM, acc, go))

    def _allgather_layout(self, pushes):
        """(buffer, rows per rank) when ``pushes`` are an 'all' mapper's full
        exchange (reference model.py:197-206): every node sends its equal
        dim-0 slab of one buffer to every other node, node k being rank k and
        each rank holding the whole buffer -- then one in-place
        ncclAllGather replaces the G(G-1) sends and receives."""
        G = self.nodes
        if self.pl.world < 2 or G != self.pl.world or len(pushes) != G * (G - 1):
            return None
        buf = pushes[0].buffer
        ext = self.buffers[buf].extent
        S, rem = divmod(ext.maxs[0], G)
        if rem or any(p.buffer != buf for p in pushes):
            return None
        if {(p.src, p.dst) for p in pushes} != {(a, b) for a in range(G) for b in range(G) if a != b}:
            return None
        for p in pushes:
            if len(p.region.boxes) != 1 or self.rank(p.src) != p.src:
                return None
            b = p.region.boxes[0]
            if b.mins != (p.src * S,) + ext.mins[1:] or b.maxs != ((p.src + 1) * S,) + ext.maxs[1:]:
                return None
        v = self.views.get((self.pl.rank, buf))
        if v is None or v.box != ext:
            return None
        return buf, S

    def _bcast_layout(self, pushes):
        """(buffer, box, root) when ``pushes`` send one box of one buffer from
        one node to every other node (e.g. an 'all' or 'fixed' read of data a
        single node wrote), node k being rank k and the box a contiguous run
        of whole rows in every rank's allocation -- then one in-place
        ncclBroadcast replaces the G-1 sends (SURVEY.md §8b cq_bcast)."""
        G = self.nodes
        if self.pl.world < 2 or G != self.pl.world or len(pushes) != G - 1:
            return None
        p0 = pushes[0]
        if len(p0.region.boxes) != 1 or self.rank(p0.src) != p0.src:
            return None
        box = p0.region.boxes[0]
        if any(p.buffer != p0.buffer or p.src != p0.src or p.region.boxes != p0.region.boxes for p in pushes):
            return None
        if {p.dst for p in pushes} != set(range(G)) - {p0.src}:
            return None
        # whole rows of the buffer: contiguous in every rank's allocation (each
        # holds the box), and decided from the plan alone, so identically on
        # every rank
        ext = self.buffers[p0.buffer].extent
        if box.mins[1:] != ext.mins[1:] or box.maxs[1:] != ext.maxs[1:]:
            return None
        return p0.buffer, box, p0.src

    def bcast(self, pushes, buf, box, root):
        """One in-place broadcast of ``box`` of ``buf`` from ``root`` on the comm stream."""
        dev = self.pl.devices[0]
        me = self.pl.rank
        v = self.views[(me, buf)]
        nbytes = box.volume() * self.buffers[buf].itemsize
        acc = [(me, buf, Region.from_box(box), me != root)]

        def go():
            N.call("cq_nccl_bcast", dev, N.STREAM_COMM, ctypes.c_void_p(v.addr(box.mins)), nbytes, root)
            STATS["bcast"] += 1
        t = self.issue(dev, N.STREAM_COMM, acc, go)
        for p in pushes:
            if self.local(p.src) or self.local(p.dst):
                self.mark_transfer(p, p.src if self.local(p.src) else p.dst, t)

    def allgather(self, pushes, buf, rows):
        """One in-place all-gather of ``buf``'s slabs on the comm stream."""
        dev = self.pl.devices[0]
        me = self.pl.rank
        v = self.views[(me, buf)]
        ext = self.buffers[buf].extent
        row_bytes = v.nbytes // ext.maxs[0]
        mine = Region.from_box(Box((me * rows,) + ext.mins[1:], ((me + 1) * rows,) + ext.maxs[1:]))
        others = Region.from_box(ext).difference(mine)
        acc = [(me, buf, mine, False), (me, buf, others, True)]

        def go():
            N.call("cq_nccl_allgather", dev, N.STREAM_COMM, ctypes.c_void_p(v.addr((me * rows,) + ext.mins[1:])),
                   ctypes.c_void_p(v.ptr), rows * row_bytes)
            STATS["allgather"] += 1
        t = self.issue(dev, N.STREAM_COMM, acc, go)
        for p in pushes:
            if self.local(p.src) or self.local(p.dst):
                self.mark_transfer(p, p.src if self.local(p.src) else p.dst, t)

    def nccl_group(self, pushes):
        """Sends and receives of this rank, posted as one NCCL group."""
        dev = self.pl.devices[0]
        accesses = []
        for p in pushes:
            if self.local(p.src):
                accesses.append((p.src, p.buffer, p.region, False))
            if self.local(p.dst):
                accesses.append((p.dst, p.buffer, p.region, True))
        staged = []

        def go():
            # pack non-contiguous boxes before the group, unpack after it
            plan_ops = []
            for p in pushes:
                eb = self.buffers[p.buffer].itemsize
                for box in p.region.boxes:
                    vol = box.volume()
                    if self.local(p.src):
                        v = self.views[(p.src, p.buffer)]
                        ptr = self._contig_ptr(v, box)
                        if ptr is None:
                            tmp = self.scratch_alloc(v.device, vol * eb)
                            N.call("cq_pack_box", v.device, N.STREAM_COMM, eb, ctypes.c_void_p(tmp),
                                   ctypes.byref(v.c), ctypes.byref(_cbox(box)))
                            ptr = tmp
                        plan_ops.append(("send", ptr, vol * eb, self.rank(p.dst)))
                    if self.local(p.dst):
                        v = self.views[(p.dst, p.buffer)]
                        ptr = self._contig_ptr(v, box)
                        if ptr is None:
                            tmp = self.scratch_alloc(v.device, vol * eb)
                            staged.append((v, tmp, box, eb))
                            ptr = tmp
                        plan_ops.append(("recv", ptr, vol * eb, self.rank(p.src)))
            STATS["nccl_groups"] += 1
            N.call("cq_nccl_group_start")
            for op, ptr, nbytes, peer in plan_ops:
                fn = "cq_nccl_send" if op == "send" else "cq_nccl_recv"
                N.call(fn, dev, N.STREAM_COMM, ctypes.c_void_p(ptr), nbytes, peer)
            N.call("cq_nccl_group_end")
            for v, tmp, box, eb in staged:
                N.call("cq_unpack_box", v.device, N.STREAM_COMM, eb, ctypes.byref(v.c),
                       ctypes.c_void_p(tmp), ctypes.byref(_cbox(box)))
        t = self.issue(dev, N.STREAM_COMM, accesses, go)
        for p in pushes:
            self.mark_transfer(p, p.src if self.local(p.src) else p.dst, t)

    def _contig_ptr(self, view, box):
        lo, hi = _pad(box)
        vlo, vhi = _pad(view.box)
        k = 0
        while k < 2 and hi[k] - lo[k] == 1:
            k += 1
        for j in range(k + 1, 3):
            if hi[j] - lo[j] != vhi[j] - vlo[j]:
                return None
        return view.addr(box.mins)

    def scratch_alloc(self, device, nbytes):
        p = ctypes.c_void_p()
        N.call("cq_malloc", device, max(nbytes, 16), ctypes.byref(p))
        self.scratch.append((device, p.value))
        return p.value

    # ---- timing marks for the trace ----------------------------------------
    def mark_transfer(self, push, node, events):
        if not self.want_trace:
            return
        start, stop = events
        if push.id is None:   # a fused block's halo transfer (fusion.HaloPush)
            self._halo_marks.append((push, node, self.dev(node), start, stop))
            return
        self.trace_marks.append((push, node, self.dev(node), start, stop))

    # ---- executes --------------------------------------------------------
    def lane(self, node):
        """Compute stream of a node: with several local nodes on one device
        (independent allocations) each gets its own lane, so their executes
        run concurrently; otherwise the compute stream."""
        lanes = self._lanes
        if lanes is None:
            lanes = self._lanes = {}
            by_dev = {}
            for n in self.local_nodes:
                by_dev.setdefault(self.dev(n), []).append(n)
            for nodes in by_dev.values():
                for i, n in enumerate(sorted(nodes)):
                    lanes[n] = N.STREAM_COMPUTE if i == 0 else N.STREAM_LANE0 + (i - 1) % N.NUM_LANES
        return lanes.get(node, N.STREAM_COMPUTE)

    def exec_command(self, cmd: ExecuteCommand, awaited):
        task = self.plan.graph.task(cmd.task_id)
        binding = self.bindings.get(task.id)
        if binding is None:
            binding = self.bindings[task.id] = bind_task(task, self.buffers)
        node, dev = cmd.node, self.dev(cmd.node)
        lane = self.lane(node)
        rviews = {}
        for a in task.accessors:
            if a.mode is AccessMode.READ:
                rviews[a.name] = self.views.get((node, a.buffer))
        wviews = {a.name: self.views[(node, a.buffer)] for a in task.writes()}
        reads = {name: (buf, reg) for name, buf, reg in cmd.reads}

        # snapshot reads of buffers this task overwrites at non-zero offsets
        for name in binding.snapshot:
            buf, reg = reads[name]
            src = rviews[name]
            bb = reg.bounding_box()
            snap = _View(node, dev, buf, bb, src.itemsize)
            self.scratch.append((dev, snap))

            def go(src=src, snap=snap, reg=reg):
                for box in reg.boxes:
                    N.call("cq_copy_box", dev, lane, src.itemsize, ctypes.byref(snap.c), dev,
                           ctypes.byref(src.c), dev, ctypes.byref(_cbox(box)))
            self.issue(dev, lane, [(node, buf, reg, False)], go)
            rviews[name] = snap

        if binding.kind == "native" and binding.args["name"] == "nbody.kick":
            pos_buf = next(a.buffer for a in task.accessors if a.name == "pos")
            if pos_buf in awaited:
                self.exec_kick(task, cmd, binding, awaited[pos_buf], dev, lane, rviews, wviews)
                return
        pieces = self.split(task, cmd, awaited)
        marks = []
        for box, dependent in pieces:
            # only a split chunk sends its halo-dependent rows to the
            # high-priority stream; an unsplit chunk stays on the compute one
            stream = N.STREAM_BOUNDARY if dependent and len(pieces) > 1 else lane
            acc = []
            for a in task.accessors:
                if a.mode is AccessMode.READ:
                    if a.name in binding.snapshot:
                        continue
                    reg = apply_mapper(a.mapper, box, task.global_range, self.buffers[a.buffer].extent)
                    acc.append((node, a.buffer, reg, False))
            for a in task.writes():
                acc.append((node, a.buffer, Region.from_box(box), True))
            t = self.issue(dev, stream, acc,
                           lambda box=box, stream=stream: self.launch(
                               binding, task, cmd, box, dev, stream, rviews, wviews, reads))
            marks.append(t)
            if self.want_trace:
                kind = binding.args["name"] if binding.kind == "native" else binding.kind
                self.launch_log.append((kind, box.volume(), dev, stream, t[0], t[1]))
        if self.want_trace:
            self.trace_marks.append((cmd, node, dev, marks, None))

    def exec_fused(self, ch, block, hostinit, replaced=()):
        """One temporally blocked wave block (fusion.py): the KL-row halo
        exchange, then per local node the interior launch (compute stream)
        and the neighbour-edge launches (boundary stream, after the
        exchange), all out of place; the alternates then become current."""
        kl = block.kl
        if hostinit:
            self.flush_group(hostinit)   # upload-time materialisation only
        ph = self._peer_halo_for(ch)
        if ph is not None:
            return self._exec_fused_peer(ch, block, replaced, ph)
        b = self.buffers[ch.a]
        self._halo_marks = []
        self.flush_group(fusion.halo_pushes(ch, kl, b.itemsize))
        if self.want_trace:
            # the plan's one-row pushes of these tasks travelled inside the
            # block's halo exchange: trace them with its times
            for p in replaced:
                for hp, node, dev, start, stop in self._halo_marks:
                    if node in (p.src, p.dst) and (hp.src, hp.dst) == (p.src, p.dst):
                        self.trace_marks.append((p, node, dev, start, stop))
                        break
        ext = _cbox(b.extent)
        W = ch.W
        ci = self.chains.index(ch)
        bi = ch.blocks.index(block)
        if self._exec_of is None:
            self._exec_of = {(c.task_id, c.node): c for c in self.plan.commands if isinstance(c, ExecuteCommand)}
        for node in sorted(ch.rows):
            if not self.local(node):
                continue
            dev = self.dev(node)
            ua, pb = self.views[(node, ch.a)], self.views[(node, ch.b)]
            oa, ob = self.alt[(node, ch.a)], self.alt[(node, ch.b)]
            marks = []
            interior, edge_t, edge_b = fusion.node_ranges(ch, node, kl)
            slots = self._amax.get((ci, node))
            # the interior reads only the node's own rows, all written by the
            # previous block's launches (ordered before it by those rows'
            # hazards), so the previous block's bound applies; the edges read
            # received halo rows and stay on the exact form
            amax_out = None if slots is None else slots + 4 * (bi + 1)
            for rng, stream in ((interior, self.lane(node)), (edge_t, N.STREAM_BOUNDARY),
                                (edge_b, N.STREAM_BOUNDARY)):
                amax_in = slots + 4 * bi if (slots is not None and bi > 0 and rng is interior) else None
                if rng is None or rng[3] <= rng[2]:
                    continue
                in_lo, in_hi, out_lo, out_hi = rng
                rin = Region.from_box(Box((in_lo, 0), (in_hi, W)))
                rout = Region.from_box(Box((out_lo, 0), (out_hi, W)))
                acc = [(ua, rin, False), (pb, rin, False), (oa, rout, True), (ob, rout, True)]

                def go(stream=stream, rng=rng, amax_in=amax_in):
                    N.call("cq_wave5_fused_bounded", dev, stream, N.KIND_CODE[b.element_kind], kl,
                           ctypes.byref(ua.c), ctypes.byref(pb.c),
                           ctypes.byref(oa.c), ctypes.byref(ob.c), rng[0], rng[1], rng[2], rng[3],
                           ctypes.byref(ext), ctypes.c_double(ch.c), ctypes.c_double(ch.k2),
                           ctypes.c_double(ch.k4), ctypes.c_void_p(amax_in), ctypes.c_void_p(amax_out))
                t = self.issue(dev, stream, acc, go)
                marks.append(t)
                if self.want_trace:
                    self.launch_log.append((f"wave5_fused{kl}", (out_hi - out_lo) * W, dev, stream, t[0], t[1]))
            # X(t+KL) / X(t+KL-1) now live in the alternates
            self.views[(node, ch.a)], self.alt[(node, ch.a)] = oa, ua
            self.views[(node, ch.b)], self.alt[(node, ch.b)] = ob, pb
            if self.want_trace:
                for i, tid in enumerate(block.tasks):
                    self.trace_marks.append((self._exec_of[(tid, node)], node, dev, marks, (i, kl)))

    def _peer_halo_for(self, ch):
        """The chain's _PeerHalo when its blocks' halo rows can go straight to
        the neighbouring ranks (one node per rank, every rank in the chain,
        the session's ``peer_halo`` -- CQ_WAVE_P2P=0 / 1 overrides it either
        way), else None; decided identically on every rank."""
        ci = self.chains.index(ch)
        if ci not in self._peer:
            env = os.environ.get("CQ_WAVE_P2P")
            allowed = env == "1" or (env != "0" and self.peer_halo)
            ok = (self.pl.world > 1 and self.nodes == self.pl.world and not self.capturing
                  and allowed
                  and getattr(N.load(), "supports_peer_memory", True)
                  and set(ch.rows) == set(range(self.nodes)) and all(self.rank(n) == n for n in ch.rows))
            ph = _PeerHalo(self, ch) if ok else None
            self._peer[ci] = ph if ph is not None and ph.ok else None
        return self._peer[ci]

    def _exec_fused_peer(self, ch, block, replaced, ph):
        """A fused block whose halo rows the neighbours wrote into this rank's
        allocation (_PeerHalo): wait for them, one launch over the slab, then
        write this rank's edge rows into the neighbours' output allocations."""
        kl = block.kl
        b = self.buffers[ch.a]
        W, me, dev, lane = ch.W, ph.me, ph.dev, self.lane(ph.me)
        ci, bi = self.chains.index(ch), ch.blocks.index(block)
        ua, pb = self.views[(me, ch.a)], self.views[(me, ch.b)]
        oa, ob = self.alt[(me, ch.a)], self.alt[(me, ch.b)]
        marks = []
        STATS["peer_blocks"] += 1
        self._halo_marks = []
        if bi == 0:
            # the chain's first halo comes through the plan's exchange
            self.flush_group(fusion.halo_pushes(ch, kl, b.itemsize))
        lo, hi = ph.lo, ph.hi
        in_lo = lo - kl if ph.top is not None else lo
        in_hi = hi + kl if ph.bot is not None else hi
        slots = self._amax.get((ci, me))
        amax_out = None if slots is None else slots + 4 * (bi + 1)
        amax_in = slots + 4 * bi if (slots is not None and bi > 0) else None
        rin = Region.from_box(Box((in_lo, 0), (in_hi, W)))
        rout = Region.from_box(Box((lo, 0), (hi, W)))
        ext = _cbox(b.extent)
        acc = [(ua, rin, False), (pb, rin, False), (oa, rout, True), (ob, rout, True)]
        # the next block's halo (up to the chain's depth) goes to the neighbours
        mir, nmir = ph.mirrors(ch.depth, (oa, ob))
        sync = ph.sync(bi)

        def go():
            # the bound covers every row read: the neighbours raised it with
            # the rows they sent before signalling (cq_peer_sync_t.peer_amax)
            N.call("cq_wave5_fused_ex", dev, lane, N.KIND_CODE[b.element_kind], kl, ctypes.byref(ua.c),
                   ctypes.byref(pb.c), ctypes.byref(oa.c), ctypes.byref(ob.c), in_lo, in_hi, lo, hi,
                   ctypes.byref(ext), ctypes.c_double(ch.c), ctypes.c_double(ch.k2), ctypes.c_double(ch.k4),
                   ctypes.c_void_p(amax_in), ctypes.c_void_p(amax_out), in_lo, in_hi, mir, nmir,
                   ctypes.byref(sync))
        t = self.issue(dev, lane, acc, go)
        marks.append(t)
        if self.want_trace:
            self.launch_log.append((f"wave5_fused{kl}", (hi - lo) * W, dev, lane, t[0], t[1]))
        pub = [t]
        self.views[(me, ch.a)], self.alt[(me, ch.a)] = oa, ua
        self.views[(me, ch.b)], self.alt[(me, ch.b)] = ob, pb
        if block is ch.blocks[-1]:
            # the neighbours' last rows into this rank land before anything
            # else here touches the halo rows
            pub.append(ph.wait(ch.depth, W, (oa, ob, ua, pb)))
        if self.want_trace:
            if self._exec_of is None:
                self._exec_of = {(c.task_id, c.node): c for c in self.plan.commands
                                 if isinstance(c, ExecuteCommand)}
            for p in replaced:
                if me not in (p.src, p.dst):
                    continue
                hm = next(((st, sp) for hp, node, _d, st, sp in self._halo_marks
                           if (hp.src, hp.dst) == (p.src, p.dst)), None)
                start, stop = hm if hm is not None else ((pub[0][0], pub[-1][1]) if p.src == me else marks[0])
                self.trace_marks.append((p, me, dev, start, stop))
            for i, tid in enumerate(block.tasks):
                self.trace_marks.append((self._exec_of[(tid, me)], me, dev, marks + pub, (i, kl)))

    def allgather_bytes(self, blob: bytes):
        """Every rank's ``blob`` (equal lengths), through one NCCL all-gather."""
        n, world, me = len(blob), self.pl.world, self.pl.rank
        dev = self.pl.devices[0]
        p = ctypes.c_void_p()
        N.call("cq_malloc", dev, n * world, ctypes.byref(p))
        host = np.frombuffer(blob, dtype=np.uint8).copy()
        out = np.empty(n * world, dtype=np.uint8)
        try:
            N.call("cq_copy_h2d", dev, N.STREAM_COMM, ctypes.c_void_p(p.value + me * n),
                   ctypes.c_void_p(host.ctypes.data), n)
            N.call("cq_nccl_allgather", dev, N.STREAM_COMM, ctypes.c_void_p(p.value + me * n), p, n)
            N.call("cq_copy_d2h", dev, N.STREAM_COMM, ctypes.c_void_p(out.ctypes.data), p, n * world)
            N.call("cq_stream_synchronize", dev, N.STREAM_COMM)
        finally:
            N.call("cq_free", dev, p)
        return [out[k * n:(k + 1) * n].tobytes() for k in range(world)]

    def exec_kick(self, task, cmd, binding, got, dev, lane, rviews, wviews):
        """The N-body kick of a chunk whose 'all'-mapped positions are partly
        still arriving (``got``: the awaited region): the j columns already
        held (cq_nbody_jcols fixed columns) run at once on the compute lane,
        the others on the boundary stream once their slabs land, and the
        finalize adds every column in column order -- the bits of one
        cq_nbody_kick, for any GPU count (reference model.py:197-206)."""
        node = cmd.node
        pos_buf = next(a.buffer for a in task.accessors if a.name == "pos")
        vbuf = next(a.buffer for a in task.accessors if a.name == "vel")
        n = self.buffers[pos_buf].extent.maxs[0]
        width = self.buffers[pos_buf].extent.maxs[1]
        if self._jcols is None:
            c = ctypes.c_int32()
            N.call("cq_nbody_jcols", ctypes.byref(c))
            self._jcols = c.value
        C = self._jcols
        box = cmd.chunk.box
        lo, hi = box.mins[0], box.maxs[0]
        runs = []   # (col_lo, col_hi, waits for the awaited slabs)
        for c in range(C):
            cols = Region.from_box(Box((n * c // C, 0), (n * (c + 1) // C, width)))
            remote = cols.overlaps(got)
            if runs and runs[-1][2] == remote and runs[-1][1] == c:
                runs[-1][1] = c + 1
            else:
                runs.append([c, c + 1, remote])
        runs.sort(key=lambda r: r[2])   # held columns first
        part = self.scratch_alloc(dev, C * (hi - lo) * 3 * 4)
        pkey = f"__kick_part_{part:x}"
        pos, vin, vout = rviews["pos"], rviews["vel_in"], wviews["vel"]
        eps2, dt = task.params["eps2"], task.params["dt"]
        marks = []
        for c0, c1, remote in runs:
            stream = N.STREAM_BOUNDARY if remote else lane
            reads = Region.from_box(Box((n * c0 // C, 0), (n * c1 // C, width)))
            acc = [(node, pos_buf, reads, False), (node, pkey, Region.from_box(Box((c0,), (c1,))), True)]

            def go(c0=c0, c1=c1, stream=stream):
                N.call("cq_nbody_kick_partial", dev, stream, ctypes.c_void_p(pos.addr((0, 0))), n,
                       ctypes.c_void_p(part), lo, hi, ctypes.c_float(eps2), c0, c1)
            t = self.issue(dev, stream, acc, go)
            marks.append(t)
            if self.want_trace:
                self.launch_log.append(("nbody.kick", box.volume() * (c1 - c0) // C, dev, stream, t[0], t[1]))
        vreg = Region.from_box(box)
        acc = [(node, pkey, Region.from_box(Box((0,), (C,))), False), (node, vbuf, vreg, False),
               (node, vbuf, vreg, True)]

        def fin():
            N.call("cq_nbody_kick_finalize", dev, lane, ctypes.c_void_p(part), ctypes.c_void_p(vin.addr((lo, 0))),
                   ctypes.c_void_p(vout.addr((lo, 0))), hi - lo, ctypes.c_float(dt))
        marks.append(self.issue(dev, lane, acc, fin))
        if self.want_trace:
            self.trace_marks.append((cmd, node, dev, marks, None))

    def split(self, task, cmd, awaited):
        """Cut the chunk along dim 0 into rows that do not read awaited
        (just-received) cells -- launched at once -- and rows that do."""
        box = cmd.chunk.box
        if not awaited or task.is_native:
            return [(box, bool(awaited))]
        lo0, hi0 = box.mins[0], box.maxs[0]
        cuts = {lo0, hi0}
        for a in task.accessors:
            if a.mode is not AccessMode.READ or a.buffer not in awaited:
                continue
            m = a.mapper
            radius = getattr(m, "radii", None)
            if radius is None and type(m).__name__ != "OneToOne":
                return [(box, True)]
            r0 = radius[0] if radius else 0
            for ab in awaited[a.buffer].boxes:
                for c in (ab.mins[0] - r0, ab.maxs[0] + r0):
                    if lo0 < c < hi0:
                        cuts.add(c)
        edges = sorted(cuts)
        out = []
        for a0, b0 in zip(edges, edges[1:]):
            sub = Box((a0,) + box.mins[1:], (b0,) + box.maxs[1:])
            dep = False
            for a in task.accessors:
                if a.mode is AccessMode.READ and a.buffer in awaited:
                    img = apply_mapper(a.mapper, sub, task.global_range, self.buffers[a.buffer].extent)
                    if img.overlaps(awaited[a.buffer]):
                        dep = True
                        break
            out.append((sub, dep))
        out.sort(key=lambda p: p[1])  # independent pieces first
        return out

    def launch(self, binding, task, cmd, box, dev, stream, rviews, wviews, reads):
        kind_name = self.buffers[task.writes()[0].buffer].element_kind
        kind = N.KIND_CODE[kind_name]
        if binding.kind == "saxpy":
            args = binding.args
            xv, yv, zv = rviews[args["x"]], rviews[args["y"]], wviews[args["out"]]
            contiguous = all(self._contig_ptr(v, box) is not None for v in (xv, yv, zv))
            aligned = kind == N.CQ_I64 or all(v.addr(box.mins) % 16 == 0 for v in (xv, yv, zv))
            if contiguous and aligned:
                alpha = args["alpha"]
                N.call("cq_saxpy", dev, stream, kind, ctypes.c_double(float(alpha)),
                       int(alpha) if kind == N.CQ_I64 else 0,
                       ctypes.c_void_p(xv.addr(box.mins)), ctypes.c_void_p(yv.addr(box.mins)),
                       ctypes.c_void_p(zv.addr(box.mins)), box.volume())
                return
            # non-contiguous chunk (n-D body on a partial range): interpreter
            binding = self.bindings.get(("expr", task.id))
            if binding is None:
                binding = self.bindings[("expr", task.id)] = _expr_binding(task, self.buffers)
        if binding.kind == "wave5":
            a = binding.args
            uacc = next(x for x in task.accessors if x.name == a["u"])
            ext = _cbox(self.buffers[uacc.buffer].extent)
            N.call("cq_wave5", dev, stream, kind, ctypes.byref(rviews[a["u"]].c),
                   ctypes.byref(rviews[a["upr"]].c), ctypes.byref(wviews[a["out"]].c),
                   ctypes.byref(_cbox(box)), ctypes.byref(ext), ctypes.c_double(a["c"]),
                   ctypes.c_double(a["k2"]), ctypes.c_double(a["k4"]))
            return
        if binding.kind == "native":
            self.launch_native(binding, task, box, dev, stream, rviews, wviews)
            return
        self.launch_expr(binding, task, cmd, box, dev, stream, rviews, wviews, reads)

    def launch_native(self, binding, task, box, dev, stream, rviews, wviews):
        name = binding.args["name"]
        lo, hi = box.mins[0], box.maxs[0]
        if name == "nbody.kick":
            pos = rviews["pos"]
            n = self.buffers[next(a.buffer for a in task.accessors if a.name == "pos")].extent.maxs[0]
            N.call("cq_nbody_kick", dev, stream, ctypes.c_void_p(pos.addr((0, 0))), n,
                   ctypes.c_void_p(rviews["vel_in"].addr((lo, 0))),
                   ctypes.c_void_p(wviews["vel"].addr((lo, 0))), lo, hi,
                   ctypes.c_float(task.params["eps2"]), ctypes.c_float(task.params["dt"]))
        elif name == "nbody.drift":
            N.call("cq_nbody_drift", dev, stream, ctypes.c_void_p(rviews["pos_in"].addr((lo, 0))),
                   ctypes.c_void_p(rviews["vel"].addr((lo, 0))),
                   ctypes.c_void_p(wviews["pos"].addr((lo, 0))), hi - lo,
                   ctypes.c_float(task.params["dt"]))
        elif name == "sgemm":
            a, b, c = rviews["a"], rviews["b"], wviews["c"]
            k = a.box.maxs[1] - a.box.mins[1]
            ncols = box.maxs[1] - box.mins[1]
            variant = {"ffma": N.SGEMM_FFMA, "3xtf32": N.SGEMM_3XTF32}.get(
                binding.args["variant"] or _default_sgemm(), N.SGEMM_FFMA)
            N.call("cq_sgemm", dev, stream, variant, ctypes.c_void_p(a.addr((lo, 0))), a.c.stride[1],
                   ctypes.c_void_p(b.addr((0, box.mins[1]))), b.c.stride[1],
                   ctypes.c_void_p(c.addr((lo, box.mins[1]))), c.c.stride[1], hi - lo, ncols, k)
        else:
            raise ValidationError(f"no native kernel '{name}'")

    def launch_expr(self, binding, task, cmd, box, dev, stream, rviews, wviews, reads):
        if binding.kind != "expr":
            binding = _expr_binding(task, self.buffers)
        kind_name = self.buffers[task.writes()[0].buffer].element_kind
        X = N.CqExpr()
        X.kind = N.KIND_CODE[kind_name]
        X.dims = task.dims
        X.box = _cbox(box)
        accs = {a.name: a for a in task.accessors}
        view_index = {}
        code_ops, code_args, consts = [], [], []
        slots = []
        X.n_out = len(binding.programs)
        kpad = 3 - task.dims
        for o, (wname, prog) in enumerate(binding.programs):
            X.out[o] = wviews[wname].c
            X.out_code_begin[o] = len(code_ops)
            base_const = len(consts)
            for v in prog.consts:
                if kind_name == "int64":
                    consts.append(int(v))
                else:
                    consts.append(int(np.float64(v).view(np.int64)))
            slot_map = {}
            for si, (acc_name, offs) in enumerate(prog.reads):
                if acc_name not in view_index:
                    vi = len(view_index)
                    view_index[acc_name] = vi
                slot_map[si] = len(slots)
                slots.append((view_index[acc_name], offs))
            for op, arg in prog.code:
                code_ops.append(op)
                if op == 0:
                    code_args.append(base_const + arg)
                elif op == 1:
                    code_args.append(kpad + arg)
                elif op == 2:
                    code_args.append(slot_map[arg])
                else:
                    code_args.append(0)
            X.out_code_end[o] = len(code_ops)
        if len(code_ops) > N.MAX_CODE or len(consts) > N.MAX_CONST or len(slots) > N.MAX_SLOTS \
                or len(view_index) > N.MAX_VIEWS:
            raise ValidationError(f"task '{task.name}': body too large for the device interpreter")
        X.n_code = len(code_ops)
        for i, (op, arg) in enumerate(zip(code_ops, code_args)):
            X.code_op[i] = op
            X.code_arg[i] = arg
        X.n_const = len(consts)
        for i, v in enumerate(consts):
            X.consts[i] = v
        X.n_slots = len(slots)
        for i, (vi, offs) in enumerate(slots):
            X.slot_view[i] = vi
            for j, o in enumerate(offs):
                X.slot_off[i][j] = o
        X.n_views = len(view_index)
        for acc_name, vi in view_index.items():
            acc = accs[acc_name]
            b = self.buffers[acc.buffer]
            X.views[vi] = rviews[acc_name].c
            X.view_extent[vi] = _cbox(b.extent)
            X.view_dims[vi] = b.dims
            # mapper check only where the clamped image may leave the region
            # (ReadView.read, model.py:442-453)
            region = reads[acc_name][1]
            need = False
            for s_vi, offs in slots:
                if s_vi != vi:
                    continue
                img = _clamped_image(box, offs, b.extent)
                if img is None or not region.contains_region(Region.from_box(img)):
                    need = True
                    break
            if need:
                if len(region.boxes) > N.MAX_CHECK:
                    raise ValidationError(f"task '{task.name}': mapped region of '{acc_name}' has "
                                          f"too many boxes for the device mapper check")
                X.view_n_check[vi] = max(1, len(region.boxes))
                if not region.boxes:
                    X.view_check[vi][0] = N.box3((0,) * b.dims, (0,) * b.dims)
                for bi, rb in enumerate(region.boxes):
                    X.view_check[vi][bi] = _cbox(rb)
        needs_check = any(X.view_n_check[vi] for vi in range(X.n_views))
        if not needs_check and jit.enabled_for(box.volume()):
            # compiled straight-line kernel (same parameter block, same bits)
            outs = [list(zip(code_ops[X.out_code_begin[o]:X.out_code_end[o]],
                             code_args[X.out_code_begin[o]:X.out_code_end[o]])) for o in range(X.n_out)]
            h = jit.handle_for(X.kind, task.dims, outs, slots, [X.view_dims[i] for i in range(X.n_views)])
            N.call("cq_jit_launch", ctypes.c_uint64(h), dev, stream, ctypes.byref(X))
            return
        N.call("cq_expr_eval", dev, stream, ctypes.byref(X))

    # ---- the walk --------------------------------------------------------
    def schedule(self):
        """Global transfer groups and per-execute awaited regions, with fused
        wave blocks substituted (identical on every rank; computed once)."""
        if self._sched is None:
            self._sched = fusion.transform(self._raw_schedule(), self.chains)
        return self._sched

    def _raw_schedule(self):
        if self._raw is not None:
            return self._raw
        # Task-major order: every push of a task depends only on commands of
        # earlier tasks (producers are read from the table state before the
        # task, scheduler.py:263-314), so all of a task's pushes can be posted
        # as ONE group before any of its executes.  That order is topological
        # -- awaits precede the executes that need them and same-task hazard
        # pushes precede the overwriting execute -- and it turns the plan's
        # per-destination push runs (e.g. an all-gather) into one NCCL group.
        segments = []
        pushes, execs, pending, cur = [], [], [], None
        for c in self.plan.commands:
            if isinstance(c, PushCommand):
                pending.append(c)
            elif isinstance(c, ExecuteCommand):
                if cur is not None and c.task_id != cur:
                    segments.append((pushes, execs))
                    pushes, execs = [], []
                cur = c.task_id
                pushes.extend(pending)
                pending = []
                execs.append(c)
        if execs or pending:
            segments.append((pushes + pending, execs))
        steps = []   # ("group", [push...]) | ("exec", cmd, awaited)
        for seg_pushes, seg_execs in segments:
            group, group_acc = [], []
            for c in seg_pushes:
                acc = [(c.src, c.buffer, c.region, False), (c.dst, c.buffer, c.region, True)]
                if any(n == n2 and b == b2 and (w or w2) and r.overlaps(r2)
                       for n, b, r, w in acc for n2, b2, r2, w2 in group_acc):
                    steps.append(("group", group))
                    group, group_acc = [], []
                group.append(c)
                group_acc.extend(acc)
            if group:
                steps.append(("group", group))
            for c in seg_execs:
                aw = {}
                for d in c.deps:
                    a = self.by_id[d]
                    if isinstance(a, AwaitPushCommand) and a.dst == c.node:
                        aw[a.buffer] = aw[a.buffer].union(a.region) if a.buffer in aw else a.region
                steps.append(("exec", c, aw))
        self._raw = steps
        return steps

    def execute(self, upload: bool = True):
        """Issue every local command of the plan (asynchronous).

        upload=True materialises host-initialised data first (node 0's copy
        and the destinations of version-1 pushes); upload=False re-runs the
        commands on the device-resident state (benchmarking)."""
        if self.t0 is None:
            if self.want_trace:
                # the trace's time origin: every stream starts after it
                for d in self.devices:
                    ev = self.event(d, timing=True)
                    N.call("cq_event_record", ctypes.c_uint64(ev), d, N.STREAM_COMPUTE)
                    self._t0[d] = ev
                    for s in N.SIDE_STREAMS:
                        N.call("cq_stream_wait_event", d, s, ctypes.c_uint64(ev))
            # untraced: no fork -- this session's ordering is its hazard
            # events, so its uploads need not wait for other sessions'
            # kernels on the shared compute stream (run_batch)
            self.t0 = dict(self._t0)
        self.uploading = upload
        if upload:
            self.seed_node0()
        for step in self.schedule():
            if step[0] == "group":
                self.flush_group(step[1])
            elif step[0] == "fused":
                self.exec_fused(*step[1:])
            elif self.local(step[1].node):
                self.exec_command(step[1], step[2])

    def _odd_chains(self):
        """Fused chains with an odd number of out-of-place blocks: one run
        leaves their current fields in the alternate allocations."""
        return [ch for ch in self.chains if len(ch.blocks) % 2]

    def _toggle_odd_chains(self):
        """Swap current and alternate allocations of the odd chains (what one
        run of them does on the device)."""
        for ch in self._odd_chains():
            for node in ch.rows:
                if self.local(node):
                    for buf in (ch.a, ch.b):
                        self.views[(node, buf)], self.alt[(node, buf)] = \
                            self.alt[(node, buf)], self.views[(node, buf)]

    def capture(self, timed: bool = False):
        """Capture one replay of the plan (``execute(upload=False)``) into a
        CUDA graph -- kernels, copies, NCCL groups and the cross-stream event
        edges -- so later replays cost one launch instead of one Python
        dispatch per command.  One local device only (the one-rank-per-GPU
        layout).  When a fused chain has an odd number of blocks, a run ends
        on the other allocations, so two graphs are captured (from either
        allocation) and ``replay`` alternates them.

        timed=True brackets every launch with event-record nodes; after each
        replay (and a synchronize) ``graph_log`` holds that replay's per-launch
        (kind, cells, device, stream, start, stop) events."""
        if len(self.devices) != 1:
            raise ValidationError("graph capture needs exactly one local device")
        d = self.devices[0]
        self.synchronize()
        self.recycle()
        self._drop_graph()
        saved = self.want_trace
        graphs, logs, events, scratch = [], [], [], []
        # a fused block swaps the current / alternate allocations as it is
        # issued; a capture failing part-way must not leave any swap behind
        views0, alt0 = dict(self.views), dict(self.alt)
        try:
            for _k in range(2 if self._odd_chains() else 1):
                self.want_trace = timed
                self.capturing = True
                N.call("cq_graph_begin", d)
                handle = ctypes.c_uint64()
                try:
                    self.execute(upload=False)
                except Exception:
                    try:
                        N.call("cq_graph_end", d, ctypes.byref(handle))
                        N.call("cq_graph_destroy", handle)
                    except NativeError:
                        pass
                    raise
                finally:
                    self.capturing = False
                    self.want_trace = saved
                N.call("cq_graph_end", d, ctypes.byref(handle))
                graphs.append(handle.value)
                # pack/unpack temporaries allocated while capturing belong to the graph
                scratch += self.scratch
                self.scratch = []
                logs.append(list(self.launch_log) if timed else [])
                if timed:
                    # the graph's event-record nodes own these events: keep them
                    # out of the recycling pool for the graph's lifetime
                    events += [ev for _d, _t, ev in self.events]
                    self.events = []
                self.recycle()  # other events recorded during capture are graph-internal
        except Exception:
            for g in graphs:
                N.call("cq_graph_destroy", ctypes.c_uint64(g))
            _free_scratch(scratch)
            for ev in events:
                N.call("cq_event_destroy", ctypes.c_uint64(ev))
            self.views.clear()
            self.views.update(views0)
            self.alt.clear()
            self.alt.update(alt0)
            self.recycle()
            raise
        # capturing executed nothing: with two graphs the views are back where
        # the device state is (the second capture started where the first ended)
        self._graph_scratch = scratch
        self.graph_events = events
        self.graphs = graphs
        self._graph_logs = logs
        self._phase = 0
        self.graph = graphs[0]
        self.graph_log = logs[0]
        return self.graph

    def _drop_graph(self):
        if self.graph:
            for d in self.devices:
                N.call("cq_stream_synchronize", d, N.STREAM_COMPUTE)
            for g in self.graphs or [self.graph]:
                N.call("cq_graph_destroy", ctypes.c_uint64(g))
            self.graph = None
        self.graphs = []
        self._graph_logs = []
        self._phase = 0
        for ev in self.graph_events:
            N.call("cq_event_destroy", ctypes.c_uint64(ev))
        self.graph_events = []
        self.graph_log = []
        _free_scratch(self._graph_scratch)

    def replay(self, times: int = 1):
        """Launch the captured graph ``times`` times (asynchronous); with two
        graphs (odd chains) they alternate and the views follow."""
        for _ in range(times):
            N.call("cq_graph_launch", ctypes.c_uint64(self.graphs[self._phase] if self.graphs else self.graph),
                   self.devices[0])
            if len(self.graphs) == 2:
                self.graph_log = self._graph_logs[self._phase]
                self._phase ^= 1
                self._toggle_odd_chains()

    def mark(self):
        """Join all streams of every local device and record a timing event
        per device on the compute stream; returns {device: event}."""
        out = {}
        for d in self.devices:
            for s in N.SIDE_STREAMS:
                ev = self.event(d)
                N.call("cq_event_record", ctypes.c_uint64(ev), d, s)
                N.call("cq_stream_wait_event", d, N.STREAM_COMPUTE, ctypes.c_uint64(ev))
            ev = self.event(d, timing=True)
            N.call("cq_event_record", ctypes.c_uint64(ev), d, N.STREAM_COMPUTE)
            for s in N.SIDE_STREAMS:
                N.call("cq_stream_wait_event", d, s, ctypes.c_uint64(ev))
            out[d] = ev
        return out

    @staticmethod
    def elapsed_ms(a, b):
        ms = ctypes.c_float()
        N.call("cq_event_elapsed_ms", ctypes.c_uint64(a), ctypes.c_uint64(b), ctypes.byref(ms))
        return ms.value

    def synchronize(self):
        for d in self.devices:
            for s in N.ALL_STREAMS:
                N.call("cq_stream_synchronize", d, s)
        self.bounce.clear()
        self.check_errors()

    def power_w(self):
        """NVML power draw per local device (watts)."""
        out = {}
        for d in self.devices:
            mw = ctypes.c_uint()
            N.call("cq_nvml_power_mw", d, ctypes.byref(mw))
            out[d] = mw.value / 1000.0
        return out

    def energy_mj(self):
        out = {}
        for d in self.devices:
            mj = ctypes.c_uint64()
            N.call("cq_nvml_energy_mj", d, ctypes.byref(mj))
            out[d] = mj.value
        return out

    def recycle(self):
        """After a synchronize: forget hazards, recycle events and traces,
        free the run's temporaries."""
        _free_scratch(self.scratch)
        self.haz = _Hazards()
        for dev, timing, ev in self.events:
            self.free_events.setdefault((dev, timing), []).append(ev)
        self.events = []
        self.trace_marks = []
        self.launch_log = []
        self.t0 = None
        self._t0 = {}

    def close(self):
        # work queued on the allocations (an exception path of run /
        # run_batch) must finish before they return to the pool
        for d in self.devices:
            for st in N.ALL_STREAMS:
                try:
                    N.call("cq_stream_synchronize", d, st)
                except NativeError:
                    pass
        self._drop_graph()
        for ph in self._peer.values():
            if ph is not None:
                ph.close()
        self._peer = {}
        self.release()
        if self._flag_host is not None:
            # back to the process-wide cache: cudaFreeHost measured 10-370 ms
            # per call, inside run_batch's timed region
            _FLAG_HOST_CACHE.setdefault(self._flag_host_bytes, []).append(self._flag_host)
            self._flag_host = None
        for pool in self.free_events.values():
            for ev in pool:
                N.call("cq_event_destroy", ctypes.c_uint64(ev))
        self.free_events = {}

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def check_errors(self):
        for d in self.devices:
            code = ctypes.c_int32()
            pt = (ctypes.c_int64 * 3)()
            N.call("cq_error_flag", d, ctypes.byref(code), pt, 1)
            _raise_flag(code.value, tuple(pt))

    def _post_error_flags(self):
        """Queue a copy of every device's error flag behind the read-back
        (``finish_results`` decodes it): a blocking read would wait for the
        copy engines, i.e. for the transfers of other runs in flight."""
        if self._flag_host is None:
            nbytes = 32 * len(self.devices)
            cached = _FLAG_HOST_CACHE.get(nbytes)
            if cached:
                ptr = cached.pop()
            else:
                ptr = ctypes.c_void_p()
                N.call("cq_host_alloc", nbytes, ctypes.byref(ptr))
            self._flag_host, self._flag_host_bytes = ptr, nbytes
        base = self._flag_host.value
        for k, d in enumerate(self.devices):
            N.call("cq_error_flag_async", d, self.d2h_stream, ctypes.c_void_p(base + 32 * k))

    def _check_posted_flags(self):
        words = (ctypes.c_uint64 * (4 * len(self.devices))).from_address(self._flag_host.value)
        for k, d in enumerate(self.devices):
            key = words[4 * k]
            if key != 0xFFFFFFFFFFFFFFFF:
                pt = tuple(ctypes.c_int64(words[4 * k + j]).value for j in (1, 2, 3))
                N.call("cq_error_flag", d, ctypes.byref(ctypes.c_int32()), (ctypes.c_int64 * 3)(), 1)  # clear
                _raise_flag(int(key & 15), pt)

    # ---- gather ------------------------------------------------------------
    def results(self, gather: str = "root", out: Optional[dict] = None):
        """Final buffers: each final piece from its lowest-id holder
        (simulator.py:210-222).  Call after ``synchronize``."""
        return self.finish_results(self.issue_results(gather, out, join=False))

    def issue_results(self, gather: str = "root", out: Optional[dict] = None, join: bool = True):
        """Post the read-back of the final buffers on the read-back stream
        (asynchronous; ``join`` first orders it after all work issued so far
        on every stream).  ``finish_results`` completes it."""
        self.gather = gather
        out_arrays = out or {}
        if gather == "none":
            return None
        if join:
            for d in self.devices:
                for st in N.ALL_STREAMS:
                    if st != self.d2h_stream:
                        ev = self.event(d)
                        N.call("cq_event_record", ctypes.c_uint64(ev), d, st)
                        N.call("cq_stream_wait_event", d, self.d2h_stream, ctypes.c_uint64(ev))
            self._post_error_flags()
        out = {}
        root = self.pl.rank == 0
        pending = []
        for name, entries in self.plan.final_locations.items():
            b = self.buffers[name]
            arr = out_arrays.get(name)
            covered = sum(r.volume() for r, _v, _h in entries) == b.extent.volume()
            if arr is None:
                arr = np.zeros(b.extent.shape, dtype=b.dtype)
            elif not covered:
                arr[...] = 0
            init_v1 = b.init.is_initialized
            for region, version, holders in entries:
                src = min(holders)
                if gather == "local":
                    # every piece this rank holds a copy of (lowest local holder)
                    mine = [h for h in holders if self.local(h)]
                    if mine:
                        src = min(mine)
                if init_v1 and version == 1:
                    if root or self.gather == "local":
                        host = self.host_array(name)
                        for box in region.boxes:
                            sl = tuple(slice(lo, hi) for lo, hi in zip(box.mins, box.maxs))
                            arr[sl] = host[sl]
                    continue
                if self.local(src) and (root or self.gather == "local"):
                    view = self.views[(src, name)]
                    pending.append((view, arr, region))
                elif self.gather == "root" and (self.local(src) or root):
                    pending.append(("nccl", src, name, arr, region))
            out[name] = arr
        direct = [p for p in pending if p[0] != "nccl"]
        temp_pins = []
        # page-lock fresh result arrays only for the copies (the caller owns
        # them afterwards), one span per array covering all its pieces;
        # `out=` arrays from pinned_empty stay pinned
        spans = {}
        for view, arr, region in direct:
            bb = region.bounding_box()
            key = id(arr)
            prev = spans.get(key)
            spans[key] = (arr, bb if prev is None else Box(
                [min(a, b) for a, b in zip(prev[1].mins, bb.mins)],
                [max(a, b) for a, b in zip(prev[1].maxs, bb.maxs)]))
        for arr, bb in spans.values():
            span = _pin_span(arr, bb, keep=False)
            if span is not None:
                temp_pins.append(span)
        bounced = []
        deferred = []   # pieces bound for pageable host memory
        st = self.d2h_stream
        for view, arr, region in direct:
            ha = N.box3((0,) * arr.ndim, arr.shape)
            for box in region.boxes:
                # a DMA into pageable memory blocks the host until the stream
                # reaches it (here: the end of the whole run), so such pieces
                # -- e.g. the halo rows a rank also holds, outside its pinned
                # output rows -- are copied by finish_results instead
                if _pin_state(*_byte_span(arr, box)) != "pinned":
                    deferred.append((view, arr, box))
                    continue
                cb = _cbox(box)
                N.call("cq_copy_box_d2h", view.device, st, view.itemsize,
                       ctypes.c_void_p(arr.ctypes.data), ctypes.byref(ha), ctypes.byref(view.c),
                       ctypes.byref(cb))
        remote = [p for p in pending if p[0] == "nccl"]
        if remote:
            if st != N.STREAM_COMM:
                raise ValidationError("gather='root' across ranks reads back on the comm stream")
            self.gather_remote(remote, bounced)
        return (out, bounced, temp_pins, root, deferred, join)

    def finish_results(self, state):
        """Wait for ``issue_results``' copies and return the buffers."""
        if state is None:
            return {}
        out, bounced, temp_pins, root, deferred, posted = state
        for d in self.devices:
            N.call("cq_stream_synchronize", d, self.d2h_stream)
        if posted:
            self._check_posted_flags()
        st = self.d2h_stream
        for view, arr, box in deferred:
            # the run is complete: pageable copies no longer wait on anything;
            # one straddling a registration edge goes through a temporary
            cb = _cbox(box)
            if _needs_bounce(arr, box):
                tmp = np.empty(box.shape, dtype=arr.dtype)
                bounced.append((arr, box, tmp))
                N.call("cq_copy_box_d2h", view.device, st, view.itemsize,
                       ctypes.c_void_p(tmp.ctypes.data), ctypes.byref(cb), ctypes.byref(view.c),
                       ctypes.byref(cb))
            else:
                N.call("cq_copy_box_d2h", view.device, st, view.itemsize,
                       ctypes.c_void_p(arr.ctypes.data), ctypes.byref(N.box3((0,) * arr.ndim, arr.shape)),
                       ctypes.byref(view.c), ctypes.byref(cb))
        if deferred:
            for d in self.devices:
                N.call("cq_stream_synchronize", d, st)
        for arr, box, tmp in bounced:
            arr[tuple(slice(lo, hi) for lo, hi in zip(box.mins, box.maxs))] = tmp
        for span in temp_pins:
            _unpin_temp(span)
        if self.gather == "root" and not root:
            return {}
        return out

    def set_inputs(self, arrays: dict):
        """Host contents of array-initialised buffers for the next
        ``execute(upload=True)`` (same shape and element kind)."""
        for name, arr in arrays.items():
            b = self.buffers[name]
            if b.init.kind != "array":
                raise ValidationError(f"buffer '{name}' is not array-initialised")
            a = np.ascontiguousarray(arr, dtype=b.dtype)
            if a.shape != b.extent.shape:
                raise ValidationError(f"buffer '{name}': input shape {a.shape} != {b.extent.shape}")
            self.host_init[name] = a
            self._overridden.add(name)
        self.pin_inputs()

    def reset_inputs(self):
        """Back to the plan's own initial contents after ``set_inputs``."""
        for name in self._overridden:
            self.host_init.pop(name, None)
        self._overridden = set()

    def gather_remote(self, items, bounced):
        """Ship final pieces held by other ranks to rank 0 over NCCL."""
        dev = self.pl.devices[0]
        ops = []
        unpack = []
        for _tag, src, name, arr, region in items:
            eb = self.buffers[name].itemsize
            for box in region.boxes:
                nbytes = box.volume() * eb
                if self.local(src):
                    v = self.views[(src, name)]
                    ptr = self._contig_ptr(v, box)
                    if ptr is None:
                        ptr = self.scratch_alloc(v.device, nbytes)
                        N.call("cq_pack_box", v.device, N.STREAM_COMM, eb, ctypes.c_void_p(ptr),
                               ctypes.byref(v.c), ctypes.byref(_cbox(box)))
                    ops.append(("send", ptr, nbytes, 0))
                else:
                    ptr = self.scratch_alloc(dev, nbytes)
                    ops.append(("recv", ptr, nbytes, self.rank(src)))
                    unpack.append((ptr, arr, box, eb))
        N.call("cq_nccl_group_start")
        for op, ptr, nbytes, peer in ops:
            fn = "cq_nccl_send" if op == "send" else "cq_nccl_recv"
            N.call(fn, dev, N.STREAM_COMM, ctypes.c_void_p(ptr), nbytes, peer)
        N.call("cq_nccl_group_end")
        for ptr, arr, box, eb in unpack:
            ha = N.box3((0,) * arr.ndim, arr.shape)
            dense = N.CqView()
            dense.ptr = ptr
            lo, hi = _pad(box)
            dense.alloc.lo[:] = lo
            dense.alloc.hi[:] = hi
            sh = [h - l for l, h in zip(lo, hi)]
            dense.stride[:] = [sh[1] * sh[2], sh[2], 1]
            cb = _cbox(box)
            if _needs_bounce(arr, box):
                tmp = np.empty(box.shape, dtype=arr.dtype)
                bounced.append((arr, box, tmp))
                N.call("cq_copy_box_d2h", dev, N.STREAM_COMM, eb, ctypes.c_void_p(tmp.ctypes.data),
                       ctypes.byref(cb), ctypes.byref(dense), ctypes.byref(cb))
                continue
            N.call("cq_copy_box_d2h", dev, N.STREAM_COMM, eb, ctypes.c_void_p(arr.ctypes.data),
                   ctypes.byref(ha), ctypes.byref(dense), ctypes.byref(cb))

    # ---- trace -------------------------------------------------------------
    def trace(self):
        """(trace events, makespan) of the commands issued since the last
        ``recycle``; times in seconds from the first ``execute``."""
        trace = []
        e0 = self.t0
        if not self.want_trace or not e0:
            return trace, Fraction(0)

        def secs(dev, ev):
            ms = ctypes.c_float()
            N.call("cq_event_elapsed_ms", ctypes.c_uint64(e0[dev]), ctypes.c_uint64(ev), ctypes.byref(ms))
            return Fraction(max(ms.value, 0.0)) / 1000

        for item in self.trace_marks:
            cmd = item[0]
            if isinstance(cmd, ExecuteCommand):
                _c, node, dev, marks, share = item
                starts = [secs(dev, a) for a, _b in marks]
                stops = [secs(dev, b) for _a, b in marks]
                if not starts:
                    continue
                t0, t1 = min(starts), max(stops)
                if share is not None:
                    # one of KL steps of a fused block: an equal slice of it
                    i, kl = share
                    t0, t1 = t0 + (t1 - t0) * i / kl, t0 + (t1 - t0) * (i + 1) / kl
                task = self.plan.graph.task(cmd.task_id)
                trace.append(TraceEvent("execute", node, cmd.id, t0, t1 - t0,
                                        frequency_ghz=cmd.frequency_ghz, task_id=cmd.task_id,
                                        task_name=task.name, label=f"{task.name}#{cmd.task_id} {cmd.chunk.box}"))
            else:
                push, node, dev, a, b = item
                t0, t1 = secs(dev, a), secs(dev, b)
                trace.append(TraceEvent("push", push.src, push.id, t0, max(t1 - t0, Fraction(0)),
                                        bytes=push.bytes,
                                        label=f"{push.buffer} {push.region} n{push.src}->n{push.dst}"))
                trace.append(TraceEvent("await_push", push.dst, push.id + 1, t1, Fraction(0),
                                        bytes=push.bytes, label=f"{push.buffer} {push.region} n{push.dst}"))
        trace.sort(key=lambda e: e.command_id)
        makespan = max((e.finish for e in trace), default=Fraction(0))
        return trace, makespan

    def release(self):
        for v in list(self.views.values()) + list(self.alt.values()):
            v.free()
        self.alt.clear()
        _free_scratch(self.scratch)
        _free_scratch(self._graph_scratch)
        _free_scratch(self._slots)
        for dev, timing, ev in self.events:
            N.call("cq_event_destroy", ctypes.c_uint64(ev))
        self.views.clear()
        self.scratch.clear()
        self.events.clear()


def _clamped_image(box, offs, extent):
    """Box of clamped read points for ``box`` shifted by ``offs`` (buffer
    axes are the leading kernel axes, model.py:442-446)."""
    lo, hi = [], []
    for j, o in enumerate(offs):
        e0, e1 = extent.mins[j], extent.maxs[j]
        a = min(max(box.mins[j] + o, e0), e1 - 1)
        b = min(max(box.maxs[j] - 1 + o, e0), e1 - 1) + 1
        if a >= b:
            return None
        lo.append(a)
        hi.append(b)
    return Box(lo, hi)


def _expr_binding(task, buffers):
    from .lowering import Binding
    from . import kernel as K
    progs = tuple((w.name, K.lower(task.body[w.name], task.params, buffers[w.buffer].element_kind))
                  for w in task.writes())
    return Binding("expr", {}, progs, frozenset())


def _default_sgemm():
    # 3xTF32 on the tensor cores meets the fp32 bar (|C - C64| / sum|a||b|
    # ~8e-8 at K = 16384) at ~5x the FFMA kernel's rate
    return os.environ.get("CQ_SGEMM", "3xtf32")


def _nvml_step(session, timeout_s: float = 1.0):
    """{device: (perf_counter time, mJ)} at the next step of each device's
    NVML energy counter.  The counter advances in coarse steps (tens of ms),
    so a run shorter than a step read between two plain reads can see no
    change at all; a window that starts and ends on a step holds exactly the
    joules of that window (its idle tail is charged at idle power by
    ``measure.measured_energy``)."""
    start = session.energy_mj()
    t0 = time.perf_counter()
    out = {}
    while len(out) < len(start):
        now_mj = session.energy_mj()
        t = time.perf_counter()
        for d, v in now_mj.items():
            if d not in out and (v != start[d] or t - t0 > timeout_s):
                out[d] = (t, v)
    return out


def run(plan: Plan, link: Optional[LinkModel] = None, *, gather: str = "root",
        out: Optional[dict] = None, trace: bool = True, energy: bool = False,
        placement: Optional[Placement] = None) -> RunResult:
    """Execute ``plan`` on B200 GPUs (drop-in for simulator.run).

    gather: "root" (default) -- rank 0 receives full buffers (single process:
            the caller gets them); "local" -- each rank fills only what it
            holds; "none" -- results stay on the devices (benchmarking).
    out:    optional {buffer: ndarray} destinations (e.g. ``pinned_empty``).
    energy: measure NVML energy per device over the run (``measured``; the
            per-task / per-device report is ``measure.measured_energy``).
    """
    if link is not None and not isinstance(link, LinkModel):
        raise ValidationError("link must be a LinkModel")
    if gather not in ("root", "local", "none"):
        raise ValidationError(f"unknown gather mode '{gather}'")
    # one-shot sessions exchange halo rows over NCCL: the peer-memory path
    # pays off in long-lived sessions (replays), while per call its setup
    # and cross-rank spin coupling cost more (profiles/r02/e2e_peer_vs_nccl_n4.txt)
    session = Session(plan, placement, trace or energy, peer_halo=False)
    try:
        e_before = idle_w = None
        if energy:
            try:
                idle_w = session.power_w()      # the devices before the run: the idle baseline
                e_before = _nvml_step(session)
            except NativeError:
                e_before = None
        session.execute(upload=True)
        session.synchronize()
        measured = {}
        if e_before is not None:
            e_after = _nvml_step(session)
            devs = {}
            for d in session.devices:
                j = (e_after[d][1] - e_before[d][1]) / 1000.0
                measured[f"energy_j_device{d}"] = j
                devs[d] = {"energy_j": j, "idle_w": idle_w[d], "window_s": e_after[d][0] - e_before[d][0]}
            measured["nvml"] = {"devices": devs,
                                "node_device": {n: session.dev(n) for n in session.local_nodes}}
        buffers = session.results(gather, out)
        events, makespan = session.trace()
    finally:
        session.close()
    return RunResult(buffers=buffers, trace=events, makespan=makespan, plan=plan, measured=measured)


def run_batch(plan: Plan, jobs, *, gather: str = "root", placement: Optional[Placement] = None,
              depth: int = 3):
    """Run ``plan`` once per job with ``depth`` executions in flight: while
    one simulation computes and another's results travel back (device->host),
    the next one's inputs travel in (host->device) -- both PCIe directions and
    the SMs work at once.  Each session uploads and reads back on its own
    streams; a session is reused once its previous read-back is complete.  Each job is ``(inputs, out)``:
    ``inputs`` {buffer: host array} (None: the plan's own initial arrays) and
    ``out`` {buffer: destination array} (None: fresh arrays; with ``out``
    arrays, a caller reusing them must give ``depth`` sets).  Returns the list
    of per-job buffer dicts, as ``run(...).buffers``; results are identical to
    calling ``run`` per job."""
    if gather not in ("root", "local", "none"):
        raise ValidationError(f"unknown gather mode '{gather}'")
    depth = max(1, min(int(depth), N.NUM_LANES // 2))
    # each session uploads and reads back on its own pair of lanes (copies of
    # different sessions then proceed concurrently on the copy engines)
    # halo rows over NCCL (run's note): with several simulations in flight the
    # peer-memory path measured batches at 1.5-2x their usual time at N=4
    sessions = [Session(plan, placement, trace=False,
                        copy_streams=(N.STREAM_LANE0 + 2 * i, N.STREAM_LANE0 + 2 * i + 1), peer_halo=False)
                for i in range(min(depth, max(1, len(jobs))))]
    if sessions[0].pl.world > 1 and gather == "root":
        for s in sessions:
            s.close()
        raise ValidationError("run_batch across ranks reads back locally: use gather='local' or 'none'")
    results = [None] * len(jobs)
    inflight = [None] * len(sessions)
    # uploads (and read-backs) of consecutive runs are chained in job order:
    # sharing the link between all runs in flight would delay the first
    # run's kernels until every queued upload is done
    chain = {}

    def follow(s, stream, key):
        for d in s.devices:
            if (key, d) in chain:
                N.call("cq_stream_wait_event", d, stream, ctypes.c_uint64(chain[(key, d)]))

    def mark(s, stream, key):
        for d in s.devices:
            ev = s.event(d)
            N.call("cq_event_record", ctypes.c_uint64(ev), d, stream)
            chain[(key, d)] = ev

    try:
        for k, (inputs, out) in enumerate(jobs):
            slot = k % len(sessions)
            s = sessions[slot]
            if inflight[slot] is not None:
                idx, state = inflight[slot]
                results[idx] = s.finish_results(state)   # also checks the run's error flags
                if state is None:   # gather="none": nothing was joined or read back
                    s.synchronize()
                    s.check_errors()
                s.recycle()
            if inputs:
                s.set_inputs(inputs)
            elif s._overridden:
                s.reset_inputs()
            follow(s, s.h2d_stream, "up")
            s.execute(upload=True)
            mark(s, s.h2d_stream, "up")
            follow(s, s.d2h_stream, "down")
            inflight[slot] = (k, s.issue_results(gather, out))
            mark(s, s.d2h_stream, "down")
        order = sorted((t for t in range(len(sessions)) if inflight[t] is not None), key=lambda t: inflight[t][0])
        for slot in order:
            idx, state = inflight[slot]
            results[idx] = sessions[slot].finish_results(state)
            sessions[slot].synchronize()
            if state is None:
                sessions[slot].check_errors()
    finally:
        for s in sessions:
            s.close()
    return results
