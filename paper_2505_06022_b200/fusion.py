"""Temporal blocking of wave ping-pong chains (an executor optimisation).

A run of consecutive tasks that all bind to the ``wave5`` fast path and
ping-pong between the same two float32 (or float64) buffers (task i+1 reads as ``u`` what
task i wrote and writes into what task i read as ``u`` -- the shape
``workloads.wave_task`` builds) is executed KL steps per HBM
pass by ``cq_wave5_fused`` instead of one ``cq_wave5`` launch per step:

* every node advances its row slab [lo, hi) from X(t), X(t-1) to X(t+KL),
  X(t+KL-1) out of place (into an alternate allocation that then becomes the
  buffer's current one);
* the interior rows [lo+KL, hi-KL) depend only on the node's own rows and
  launch at once; the KL rows next to a neighbour need the neighbour's KL
  nearest rows of X(t) and X(t-1), exchanged once per block (NCCL / DMA,
  through the executor's ordinary transfer path) while the interior runs --
  or, with one node per rank, stored into the neighbour's memory by the
  previous block's pass itself (executor._PeerHalo, one launch per block);
* each cell is the same DSL tree with the same operands as the per-step
  execution, so results are bit-identical (tests/test_gpu_parity.py).

What changes against executing the plan command by command: the plan's
one-row halo pushes of the fused tasks are replaced by one KL-row exchange
per block; the last task's pushes are still posted after the chain, so every
halo row the plan's ``final_locations`` lists holds its final version.
Chains run as many KL = 8 blocks as fit (half the bytes per step of KL = 4)
and one KL = 4 block, placed first, for a remaining quarter (``_blocks``;
100 steps = 1 x KL4 + 12 x KL8).  An odd number of out-of-place blocks
leaves a run's fields in the alternate allocations: the executor follows
them, and a CUDA-graph capture records two alternating graphs
(``Session.capture``).  Leftover steps (< 4) run one step at a time.

``CQ_WAVE_FUSE=0`` disables the transformation.
"""

import os
from dataclasses import dataclass, field

from .lowering import bind_task
from .region import Box, Region

KL_BASE = 4
KL_PARITY = 8
MIN_ROWS = 4 * KL_PARITY   # slab height below which a node's chain is not fused
MIN_CHAIN = 2 * KL_BASE


def enabled() -> bool:
    return os.environ.get("CQ_WAVE_FUSE", "1") != "0"


@dataclass
class Block:
    tasks: tuple       # task ids, in order
    kl: int


@dataclass
class Chain:
    a: str             # buffer holding X(t) at every block start (read as u)
    b: str             # buffer holding X(t-1)
    c: float
    k2: float
    k4: float
    H: int
    W: int
    rows: dict         # node -> (lo, hi)
    blocks: list       # [Block]
    plain: tuple       # task ids run one step at a time after the blocks
    last_pushes: list = field(default_factory=list)  # plan pushes of the last task

    @property
    def depth(self) -> int:
        return max(b.kl for b in self.blocks)

    def fused_tasks(self):
        return {t for b in self.blocks for t in b.tasks}


@dataclass(frozen=True)
class HaloPush:
    """A transfer the fused execution adds (KL-row halo), not a plan command:
    the transfer path treats it like a PushCommand; it has no trace id."""
    src: int
    dst: int
    buffer: str
    region: Region
    element_bytes: int
    deps: tuple = (None,)
    id: object = None

    @property
    def bytes(self) -> int:
        return self.region.volume() * self.element_bytes


def _task_segments(steps):
    """task id -> (pushes of its groups, execs), from the executor schedule
    (each group belongs to the task of the next execute step)."""
    seg = {}
    pending = []
    for st in steps:
        if st[0] == "group":
            pending.extend(st[1])
        else:
            cmd = st[1]
            p, e = seg.setdefault(cmd.task_id, ([], []))
            p.extend(pending)
            pending = []
            e.append(cmd)
    if pending and seg:
        last = max(seg)
        seg[last][0].extend(pending)
    return seg


def _wave_info(task, buffers):
    """(u buffer, upr buffer, c, k2, k4, H, W) when the task is a float32
    ping-pong wave step on the fused kernel's terms, else None."""
    if task.is_native or task.dims != 2:
        return None
    b = bind_task(task, buffers)
    if b.kind != "wave5":
        return None
    acc = {a.name: a for a in task.accessors}
    ubuf, pbuf, obuf = acc[b.args["u"]].buffer, acc[b.args["upr"]].buffer, acc[b.args["out"]].buffer
    if obuf != pbuf or ubuf == pbuf:
        return None
    bu, bp = buffers[ubuf], buffers[pbuf]
    if bu.element_kind not in ("float32", "float64") or bp.element_kind != bu.element_kind \
            or bu.extent != bp.extent:
        return None
    if b.args["k2"] != 2.0 or b.args["k4"] != 4.0:
        return None   # the fused kernel forms 2u and 4u as exact sums
    ext = bu.extent
    if ext.mins != (0, 0) or task.global_range != ext:
        return None
    H, W = ext.maxs
    if W % 4:
        return None
    return ubuf, pbuf, b.args["c"], b.args["k2"], b.args["k4"], H, W


def _slabs(execs, H, W):
    """node -> (lo, hi) when the executes are full-width row slabs tiling [0, H)."""
    rows = {}
    for c in execs:
        box = c.chunk.box
        if box.mins[1] != 0 or box.maxs[1] != W or c.node in rows:
            return None
        rows[c.node] = (box.mins[0], box.maxs[0])
    spans = sorted(rows.values())
    if not spans or spans[0][0] != 0 or spans[-1][1] != H:
        return None
    if any(a[1] != b[0] for a, b in zip(spans, spans[1:])):
        return None
    return rows


def _halo_pushes_ok(pushes, ubuf, rows, W):
    """The non-host-initialised pushes of a task are exactly one-row halos
    of its u buffer between neighbouring slabs."""
    for p in pushes:
        if not p.deps:
            continue
        if p.buffer != ubuf or len(p.region.boxes) != 1:
            return False
        box = p.region.boxes[0]
        if box.maxs[0] - box.mins[0] != 1 or box.mins[1] != 0 or box.maxs[1] != W:
            return False
        r = box.mins[0]
        slo, shi = rows[p.src]
        dlo, dhi = rows[p.dst]
        if not ((r == slo and dhi == slo) or (r == shi - 1 and dlo == shi)):
            return False
    return True


def _blocks(tids, kind="float32"):
    """Split a chain into out-of-place blocks: as many KL=8 blocks as fit
    (KL=8 moves half the bytes per step of KL=4) and a KL=4 block for a
    remaining quarter, placed first -- a run's first block has no magnitude
    bound and keeps the exact form, which costs the HBM-bound 4-step pass
    nothing but the FP-bound 8-step pass ~15% (cq_wave5_fused_bounded).  An
    odd block count leaves a run's fields in the alternate allocations; the
    executor follows them, and graph capture then records two alternating
    graphs.  Tasks left over (< 4) run plain."""
    q, _r = divmod(len(tids), KL_BASE)   # quarter blocks
    sizes = [KL_BASE] * (q % 2) + [KL_PARITY] * (q // 2)
    if not sizes:
        return [], tuple(tids)
    blocks, i = [], 0
    for kl in sizes:
        blocks.append(Block(tuple(tids[i:i + kl]), kl))
        i += kl
    return blocks, tuple(tids[i:])


def find_chains(plan, steps):
    """Fusable wave chains of ``plan`` (deterministic: every rank agrees)."""
    if not enabled():
        return []
    graph = plan.graph
    buffers = graph.buffers
    seg = _task_segments(steps)
    chains = []
    cur = None   # (info, rows, [tids])

    def close():
        if cur is None:
            return
        info, rows, tids = cur
        if len(tids) < MIN_CHAIN:
            return
        blocks, plain = _blocks(tids, buffers[info[0]].element_kind)
        if not blocks:
            return
        u0, p0, c, k2, k4, H, W = info
        chains.append(Chain(u0, p0, c, k2, k4, H, W, rows, blocks, plain,
                            [p for p in seg[tids[-1]][0] if p.deps]))

    for tid in sorted(seg):
        pushes, execs = seg[tid]
        task = graph.task(tid)
        info = _wave_info(task, buffers)
        rows = _slabs(execs, info[5], info[6]) if info else None
        ok = (info is not None and rows is not None
              and all(hi - lo >= MIN_ROWS for lo, hi in rows.values())
              and _halo_pushes_ok(pushes, info[0], rows, info[6]))
        if ok and cur is not None:
            pinfo, prows, ptids = cur
            ptask_u, ptask_p = _task_buffers(graph.task(ptids[-1]), buffers)
            cont = (info[0] == ptask_p and info[1] == ptask_u and info[2:] == pinfo[2:] and rows == prows)
            if cont:
                ptids.append(tid)
                continue
        close()
        cur = (info, rows, [tid]) if ok else None
    close()
    return chains


def _task_buffers(task, buffers):
    info = _wave_info(task, buffers)
    return info[0], info[1]


def transform(steps, chains):
    """Replace the steps of every fused block by one ("fused", chain, block,
    host-init pushes, plan pushes the block's exchange replaces) step; after a chain whose last task is fused, post that
    task's plan pushes (so the final halo rows hold their final versions)."""
    if not chains:
        return steps
    block_of = {}
    for ch in chains:
        for bl in ch.blocks:
            for t in bl.tasks:
                block_of[t] = (ch, bl)
    # task of each step (groups belong to the next execute's task)
    owner = [None] * len(steps)
    nxt = None
    for i in range(len(steps) - 1, -1, -1):
        if steps[i][0] == "exec":
            nxt = steps[i][1].task_id
        owner[i] = nxt
    out = []
    emitted = set()
    hostinit = {}
    replaced = {}
    for i, st in enumerate(steps):
        t = owner[i]
        if t is None and st[0] == "group":
            # trailing pushes after the last execute: keep
            out.append(st)
            continue
        hit = block_of.get(t)
        if hit is None:
            out.append(st)
            continue
        ch, bl = hit
        key = (id(ch), bl.tasks[0])
        if st[0] == "group":
            hostinit.setdefault(key, []).extend(p for p in st[1] if not p.deps)
            posted_later = set(map(id, ch.last_pushes)) if not ch.plain else set()
            replaced.setdefault(key, []).extend(p for p in st[1] if p.deps and id(p) not in posted_later)
        if key not in emitted:
            emitted.add(key)
            out.append(("fused", ch, bl, hostinit.setdefault(key, []), replaced.setdefault(key, [])))
        if st[0] == "exec" and not ch.plain and t == ch.blocks[-1].tasks[-1] \
                and _is_last_exec(steps, i, t):
            if ch.last_pushes:
                out.append(("group", list(ch.last_pushes)))
    return out


def _is_last_exec(steps, i, t):
    for st in steps[i + 1:]:
        if st[0] == "exec":
            return st[1].task_id != t
    return True


def node_ranges(chain, node, kl):
    """(interior, top edge, bottom edge) launches of ``node`` for a block of
    depth ``kl``: each (in_lo, in_hi, out_lo, out_hi) or None."""
    lo, hi = chain.rows[node]
    H = chain.H
    top = lo > 0
    bot = hi < H
    interior = (lo, hi, lo + kl if top else lo, hi - kl if bot else hi)
    edge_t = (lo - kl, min(hi, lo + 2 * kl), lo, lo + kl) if top else None
    edge_b = (max(lo, hi - 2 * kl), hi + kl, hi - kl, hi) if bot else None
    return interior, edge_t, edge_b


def halo_pushes(chain, kl, itemsize):
    """The KL-row exchange of a block: every node sends its KL rows nearest
    to each neighbour, of both X(t) and X(t-1)."""
    W = chain.W
    by_lo = {lo: n for n, (lo, _hi) in chain.rows.items()}
    by_hi = {hi: n for n, (_lo, hi) in chain.rows.items()}
    out = []
    for n in sorted(chain.rows):
        lo, hi = chain.rows[n]
        for buf in (chain.a, chain.b):
            if lo > 0:
                up = by_hi[lo]
                out.append(HaloPush(n, up, buf, Region.from_box(Box((lo, 0), (lo + kl, W))), itemsize))
            if hi < chain.H:
                down = by_lo[hi]
                out.append(HaloPush(n, down, buf, Region.from_box(Box((hi - kl, 0), (hi, W))), itemsize))
    return out


__all__ = ["Chain", "Block", "HaloPush", "find_chains", "transform", "node_ranges", "halo_pushes", "enabled"]
