"""A numpy test double of libcq (include/cq.h) for CPU-only tests.

TEST INFRASTRUCTURE ONLY.  It lets the executor's host logic -- allocation,
Kahn-order walk, transfer grouping, NCCL send/recv matching, hazard events,
interior/boundary splitting, snapshots, the packed CqExpr struct, gather --
run without a GPU, including a 2-rank torch.distributed *gloo* run where
the NCCL group ops travel over gloo.  Kernels are plain numpy with the same
per-operator rounding; the real kernels are tested on the B200 by
tests/test_gpu_parity.py.  Installed by monkeypatching ``_native._lib``.
"""

import ctypes

import numpy as np

from paper_2505_06022_b200 import _native as N

_DT = {N.CQ_F64: np.float64, N.CQ_F32: np.float32, N.CQ_I64: np.int64}


def _val(x):
    return x.value if hasattr(x, "value") else x


def _obj(x):
    return x._obj if hasattr(x, "_obj") else x


class FakeLib:
    # no CUDA IPC between the gloo test processes: fused chains across ranks
    # take the NCCL halo exchange (the peer-memory path is covered on GPUs)
    supports_peer_memory = False

    def __init__(self, ndev=1, transport=None):
        self.ndev = ndev
        self.blocks = {}      # base -> np.uint8 array
        self.next = 1 << 44
        self.err = b""
        self.transport = transport
        self.group = None
        self.flag = None
        self.launches = []
        self.events = 0

    # ----------------------------------------------------------- memory
    def _mem(self, addr, nbytes):
        for base, blk in self.blocks.items():
            if base <= addr < base + blk.size:
                off = addr - base
                assert off + nbytes <= blk.size, "device access out of bounds"
                return blk[off:off + nbytes]
        buf = (ctypes.c_uint8 * nbytes).from_address(addr)
        return np.ctypeslib.as_array(buf)

    def _arr(self, addr, shape, strides_elems, dtype):
        dtype = np.dtype(dtype)
        n = 1 + sum((s - 1) * st for s, st in zip(shape, strides_elems)) if all(shape) else 0
        raw = self._mem(addr, n * dtype.itemsize)
        flat = raw.view(dtype)
        return np.lib.stride_tricks.as_strided(flat, shape=shape,
                                               strides=[s * dtype.itemsize for s in strides_elems])

    def _view(self, v, dtype, box=None):
        """ndarray over the cells of ``box`` (global coords) of view ``v``."""
        lo = list(v.alloc.lo)
        box = box or v.alloc
        off = sum((box.lo[k] - lo[k]) * v.stride[k] for k in range(3))
        shape = [box.hi[k] - box.lo[k] for k in range(3)]
        dt = np.dtype(dtype)
        return self._arr(v.ptr + off * dt.itemsize, shape, list(v.stride), dt)

    def _host(self, addr, alloc, box, dtype):
        sh = [alloc.hi[k] - alloc.lo[k] for k in range(3)]
        st = [sh[1] * sh[2], sh[2], 1]
        off = sum((box.lo[k] - alloc.lo[k]) * st[k] for k in range(3))
        dt = np.dtype(dtype)
        return self._arr(addr + off * dt.itemsize, [box.hi[k] - box.lo[k] for k in range(3)], st, dt)

    @staticmethod
    def _eb(eb):
        return {4: np.uint32, 8: np.uint64, 1: np.uint8, 2: np.uint16}[eb]

    # ----------------------------------------------------------- runtime
    def cq_last_error(self):
        return self.err

    def cq_version(self, p):
        _obj(p).value = 1
        return 0

    def cq_device_count(self, p):
        _obj(p).value = self.ndev
        return 0

    def cq_init_device(self, d):
        return 0

    def cq_device_props(self, d, sm, l2, clk, mem):
        _obj(sm).value, _obj(l2).value, _obj(clk).value, _obj(mem).value = 148, 126 << 20, 1965000, 180 << 30
        return 0

    def cq_enable_peer(self, d, p, en):
        _obj(en).value = 1
        return 0

    def cq_shutdown(self):
        return 0

    def cq_malloc(self, d, nbytes, p):
        n = int(_val(nbytes))
        base = self.next
        self.next += ((n + (1 << 20)) >> 20 << 20) + (1 << 20)
        self.blocks[base] = np.zeros(max(n, 1), np.uint8)
        _obj(p).value = base
        return 0

    def cq_free(self, d, p):
        self.blocks.pop(_val(p), None)
        return 0

    def cq_pool_trim(self, d):
        return 0

    def cq_host_register(self, p, n):
        return 0

    def cq_host_unregister(self, p):
        return 0

    def cq_copy_h2d(self, d, s, dst, src, n):
        n = int(_val(n))
        self._mem(_val(dst), n)[:] = self._mem(_val(src), n)
        return 0

    cq_copy_d2h = cq_copy_h2d

    def cq_copy_box(self, d, s, eb, dst, dd, src, sd, box):
        dt = self._eb(eb)
        b = _obj(box)
        self._view(_obj(dst), dt, b)[...] = self._view(_obj(src), dt, b)
        return 0

    def cq_copy_box_h2d(self, d, s, eb, dst, host, halloc, box):
        dt = self._eb(eb)
        b = _obj(box)
        self._view(_obj(dst), dt, b)[...] = self._host(_val(host), _obj(halloc), b, dt)
        return 0

    def cq_copy_box_d2h(self, d, s, eb, host, halloc, src, box):
        dt = self._eb(eb)
        b = _obj(box)
        self._host(_val(host), _obj(halloc), b, dt)[...] = self._view(_obj(src), dt, b)
        return 0

    def cq_pack_box(self, d, s, eb, dense, src, box):
        dt = self._eb(eb)
        b = _obj(box)
        self._host(_val(dense), b, b, dt)[...] = self._view(_obj(src), dt, b)
        return 0

    def cq_unpack_box(self, d, s, eb, dst, dense, box):
        dt = self._eb(eb)
        b = _obj(box)
        self._view(_obj(dst), dt, b)[...] = self._host(_val(dense), b, b, dt)
        return 0

    def cq_event_create(self, d, timing, p):
        self.events += 1
        _obj(p).value = self.events
        return 0

    def cq_event_destroy(self, e):
        return 0

    def cq_event_record(self, e, d, s):
        return 0

    def cq_event_record_timed(self, e, d, s):
        return 0

    def cq_stream_wait_event(self, d, s, e):
        return 0

    def cq_event_synchronize(self, e):
        return 0

    def cq_event_elapsed_ms(self, a, b, p):
        _obj(p).value = 0.001 * (_val(b) - _val(a))
        return 0

    def cq_stream_synchronize(self, d, s):
        return 0

    def cq_device_synchronize(self, d):
        return 0

    # -------------------------------------------------------------- NCCL
    def cq_nccl_unique_id(self, buf):
        return 0

    def cq_nccl_init(self, d, n, r, uid):
        return 0

    def cq_nccl_group_start(self):
        self.group = []
        return 0

    def cq_nccl_group_end(self):
        ops, self.group = self.group, None
        self.transport.exchange(ops, self)
        return 0

    def cq_nccl_send(self, d, s, buf, n, peer):
        self.group.append(("send", _val(buf), int(_val(n)), int(_val(peer))))
        return 0

    def cq_nccl_recv(self, d, s, buf, n, peer):
        self.group.append(("recv", _val(buf), int(_val(n)), int(_val(peer))))
        return 0

    def cq_nccl_allgather(self, d, s, send, recv, n):
        """In-place ncclAllGather semantics over the transport."""
        self.transport.allgather(self, _val(send), _val(recv), int(_val(n)))
        self.launches.append(("allgather", int(_val(n))))
        return 0

    def cq_nccl_bcast(self, d, s, buf, n, root):
        """In-place ncclBroadcast semantics over the transport."""
        self.transport.bcast(self, _val(buf), int(_val(n)), int(_val(root)))
        self.launches.append(("bcast", int(_val(n))))
        return 0

    def cq_nccl_destroy(self):
        return 0

    # ----------------------------------------------------------- kernels
    def cq_fill(self, d, s, kind, dst, box, ext, mode, val, ival):
        dt = _DT[kind]
        b, e = _obj(box), _obj(ext)
        out = self._view(_obj(dst), dt, b)
        if mode == 1:
            e1, e2 = e.hi[1] - e.lo[1], e.hi[2] - e.lo[2]
            i0, i1, i2 = np.meshgrid(*[np.arange(b.lo[k], b.hi[k]) for k in range(3)], indexing="ij")
            out[...] = ((i0 * e1 + i1) * e2 + i2).astype(dt)
        elif mode == 2:
            out[...] = ival if kind == N.CQ_I64 else dt(_val(val))
        else:
            out[...] = 0
        return 0

    def cq_saxpy(self, d, s, kind, alpha, ialpha, x, y, z, n):
        dt = _DT[kind]
        n = int(_val(n))
        xa = self._arr(_val(x), [n], [1], dt)
        ya = self._arr(_val(y), [n], [1], dt)
        za = self._arr(_val(z), [n], [1], dt)
        a = np.int64(ialpha) if kind == N.CQ_I64 else dt(_val(alpha))
        with np.errstate(all="ignore"):
            za[...] = (a * xa).astype(dt) + ya
        self.launches.append("saxpy")
        return 0

    def cq_wave5(self, d, s, kind, u, upr, out, box, ext, c, k2, k4):
        dt = _DT[kind]
        u, upr, out, b, e = (_obj(x) for x in (u, upr, out, box, ext))
        H, W = e.hi[1], e.hi[2]
        rows = np.arange(b.lo[1], b.hi[1])
        cols = np.arange(b.lo[2], b.hi[2])
        uu = self._view(u, dt)
        lo1, lo2 = u.alloc.lo[1], u.alloc.lo[2]

        def at(r, cc):
            return uu[0][np.clip(r, 0, H - 1)[:, None] - lo1, np.clip(cc, 0, W - 1)[None, :] - lo2]
        cc = at(rows, cols)
        c, k2, k4 = dt(_val(c)), dt(_val(k2)), dt(_val(k4))
        lap = (((at(rows - 1, cols) + at(rows + 1, cols)) + at(rows, cols - 1)) + at(rows, cols + 1)) - k4 * cc
        res = ((k2 * cc) - self._view(upr, dt, b)[0]) + c * lap
        self._view(out, dt, b)[0][...] = res
        self.launches.append("wave5")
        return 0

    def cq_wave5_fused_bounded(self, d, s, kind, levels, u, upr, out_last, out_prev, in_lo, in_hi, out_lo, out_hi,
                               ext, c, k2, k4, amax_in, amax_out):
        # the bound only selects an equivalent arithmetic form on the GPU
        self.fused_bounds = getattr(self, "fused_bounds", [])
        self.fused_bounds.append((_val(amax_in), _val(amax_out)))
        return self.cq_wave5_fused(d, s, kind, levels, u, upr, out_last, out_prev, in_lo, in_hi, out_lo, out_hi,
                                   ext, c, k2, k4)

    def cq_wave5_fused(self, d, s, kind, levels, u, upr, out_last, out_prev, in_lo, in_hi, out_lo, out_hi, ext, c,
                       k2, k4):
        """KL ping-pong steps on rows [in_lo, in_hi) (edge rows replicate,
        which is exact at the true borders and only spoils rows outside the
        trapezoid), then rows [out_lo, out_hi) of the last two levels."""
        u, upr, ol, op, e = (_obj(x) for x in (u, upr, out_last, out_prev, ext))
        in_lo, in_hi, out_lo, out_hi, levels = (_val(x) for x in (in_lo, in_hi, out_lo, out_hi, levels))
        dt = _DT[_val(kind)]
        W = e.hi[2]
        box = N.box3((in_lo, 0), (in_hi, W))
        cur = self._view(u, dt, box)[0].copy()
        prev = self._view(upr, dt, box)[0].copy()
        c, k2, k4 = dt(_val(c)), dt(_val(k2)), dt(_val(k4))
        cols = np.arange(W)
        for _ in range(levels):
            n = cur[np.clip(np.arange(cur.shape[0]) - 1, 0, cur.shape[0] - 1)]
            sth = cur[np.clip(np.arange(cur.shape[0]) + 1, 0, cur.shape[0] - 1)]
            w = cur[:, np.clip(cols - 1, 0, W - 1)]
            east = cur[:, np.clip(cols + 1, 0, W - 1)]
            lap = (((n + sth) + w) + east) - k4 * cur
            cur, prev = ((k2 * cur) - prev) + c * lap, cur
        ob = N.box3((out_lo, 0), (out_hi, W))
        self._view(ol, dt, ob)[0][...] = cur[out_lo - in_lo:out_hi - in_lo]
        self._view(op, dt, ob)[0][...] = prev[out_lo - in_lo:out_hi - in_lo]
        self.launches.append("wave5_fused")
        return 0

    def cq_expr_eval(self, d, s, X):
        X = _obj(X)
        dt = _DT[X.kind]
        b = X.box
        p = np.meshgrid(*[np.arange(b.lo[k], b.hi[k], dtype=np.int64) for k in range(3)], indexing="ij")
        shape = p[0].shape
        results = []
        for o in range(X.n_out):
            stack = []
            for pc in range(X.out_code_begin[o], X.out_code_end[o]):
                op, arg = X.code_op[pc], X.code_arg[pc]
                if op == 0:
                    bits = np.int64(X.consts[arg])
                    v = bits if X.kind == N.CQ_I64 else bits.view(np.float64)
                    stack.append(np.full(shape, v).astype(dt))
                elif op == 1:
                    stack.append(p[arg].astype(dt))
                elif op == 2:
                    vi = X.slot_view[arg]
                    bd = X.view_dims[vi]
                    ext = X.view_extent[vi]
                    q = [np.zeros(shape, np.int64) for _ in range(3)]
                    for j in range(bd):
                        ax = 3 - bd + j
                        q[ax] = np.clip(p[3 - X.dims + j] + X.slot_off[arg][j], ext.lo[ax], ext.hi[ax] - 1)
                    if X.view_n_check[vi] > 0:
                        inside = np.zeros(shape, bool)
                        for bi in range(X.view_n_check[vi]):
                            cb = X.view_check[vi][bi]
                            inside |= np.all([(q[k] >= cb.lo[k]) & (q[k] < cb.hi[k]) for k in range(3)], axis=0)
                        if not inside.all():
                            self.flag = N.CQ_ERR_MAPPER
                            return 0
                    v = X.views[vi]
                    arr = self._view(v, dt)
                    stack.append(arr[q[0] - v.alloc.lo[0], q[1] - v.alloc.lo[1], q[2] - v.alloc.lo[2]])
                elif op == 3:
                    with np.errstate(all="ignore"):
                        stack[-1] = (-stack[-1]).astype(dt)
                else:
                    bb = stack.pop()
                    aa = stack.pop()
                    with np.errstate(all="ignore"):
                        if op == 4:
                            r = aa + bb
                        elif op == 5:
                            r = aa - bb
                        elif op == 6:
                            r = aa * bb
                        elif X.kind == N.CQ_I64:
                            if np.any(bb == 0):
                                self.flag = N.CQ_ERR_EVAL
                                return 0
                            q = np.abs(aa.astype(np.float64)) // np.abs(bb.astype(np.float64))
                            r = np.where((aa < 0) != (bb < 0), -q, q).astype(np.int64)
                        else:
                            r = aa / bb
                    stack.append(r.astype(dt))
            results.append(stack[0])
        for o in range(X.n_out):
            self._view(X.out[o], dt, b)[...] = results[o]
        self.launches.append("expr")
        return 0

    def cq_jit_compile(self, *args):
        # real NVRTC compile of the generated kernel (host-only, no GPU);
        # the double then runs the body through its interpreter
        self.jit_compiled = getattr(self, "jit_compiled", 0) + 1
        status = N.load_host().cq_jit_compile(*args)
        if status:
            self.err = N.load_host().cq_last_error()
        return status

    def cq_jit_launch(self, h, d, s, X):
        self.launches.append("jit")
        return self.cq_expr_eval(d, s, X)

    def cq_host_alloc(self, nbytes, p):
        buf = np.zeros(int(_val(nbytes)), dtype=np.uint8)
        self.host_bufs = getattr(self, "host_bufs", {})
        self.host_bufs[buf.ctypes.data] = buf
        _obj(p).value = buf.ctypes.data
        return 0

    def cq_host_free(self, p):
        getattr(self, "host_bufs", {}).pop(_val(p), None)
        return 0

    def cq_error_flag_async(self, d, s, host):
        words = (ctypes.c_uint64 * 4).from_address(_val(host))
        words[0] = 0xFFFFFFFFFFFFFFFF if not self.flag else self.flag
        words[1] = words[2] = words[3] = 0
        return 0

    def cq_error_flag(self, d, code, pt, clear):
        _obj(code).value = self.flag or 0
        if clear:
            self.flag = None
        return 0

    NB_JCOLS = 8

    def cq_nbody_jcols(self, p):
        _obj(p).value = self.NB_JCOLS
        return 0

    def cq_nbody_kick_partial(self, d, s, pos, n, part, lo, hi, eps2, c0, c1):
        """Per-column partial accelerations (float64 sums rounded once) --
        the structure, not the bits, of the GPU kernel."""
        n, lo, hi, c0, c1 = (int(_val(x)) for x in (n, lo, hi, c0, c1))
        C = self.NB_JCOLS
        P = self._arr(_val(pos), [n, 4], [4, 1], np.float32).astype(np.float64)
        out = self._arr(_val(part), [C, hi - lo, 3], [(hi - lo) * 3, 3, 1], np.float32)
        for c in range(c0, c1):
            jb, je = n * c // C, n * (c + 1) // C
            d3 = P[None, jb:je, :3] - P[lo:hi, None, :3]
            r2 = (d3 ** 2).sum(-1) + _val(eps2)
            out[c] = (d3 * (P[None, jb:je, 3] / r2 ** 1.5)[..., None]).sum(1).astype(np.float32)
        self.launches.append("nbody.partial")
        return 0

    def cq_nbody_kick_finalize(self, d, s, part, vin, vout, count, dt_):
        count = int(_val(count))
        C = self.NB_JCOLS
        pa = self._arr(_val(part), [C, count, 3], [count * 3, 3, 1], np.float32)
        acc = np.zeros((count, 3), np.float32)
        for c in range(C):
            acc += pa[c]
        vi = self._arr(_val(vin), [count, 4], [4, 1], np.float32)
        res = vi.copy()
        res[:, :3] += np.float32(_val(dt_)) * acc
        self._arr(_val(vout), [count, 4], [4, 1], np.float32)[...] = res
        return 0

    def cq_nbody_kick(self, d, s, pos, n, vin, vout, lo, hi, eps2, dt_):
        lo, hi = int(_val(lo)), int(_val(hi))
        part = np.zeros((self.NB_JCOLS, hi - lo, 3), np.float32)
        addr = part.ctypes.data
        self.cq_nbody_kick_partial(d, s, pos, n, addr, lo, hi, eps2, 0, self.NB_JCOLS)
        self.cq_nbody_kick_finalize(d, s, addr, vin, vout, hi - lo, dt_)
        return 0

    def cq_nbody_drift(self, d, s, pin, v, pout, count, dt_):
        count = int(_val(count))
        a = self._arr(_val(pin), [count, 4], [4, 1], np.float32).copy()
        b = self._arr(_val(v), [count, 4], [4, 1], np.float32)
        a[:, :3] += np.float32(_val(dt_)) * b[:, :3]
        self._arr(_val(pout), [count, 4], [4, 1], np.float32)[...] = a
        return 0

    def cq_sgemm(self, d, s, variant, a, lda, b, ldb, c, ldc, m, n, k):
        m, n, k = int(_val(m)), int(_val(n)), int(_val(k))
        A = self._arr(_val(a), [m, k], [int(_val(lda)), 1], np.float32)
        B = self._arr(_val(b), [k, n], [int(_val(ldb)), 1], np.float32)
        self._arr(_val(c), [m, n], [int(_val(ldc)), 1], np.float32)[...] = \
            (A.astype(np.float64) @ B.astype(np.float64)).astype(np.float32)
        return 0

    # -------------------------------------------------------------- NVML
    def _nvml_absent(self, *a):
        self.err = b"NVML not available in the CPU test double"
        return N.CQ_ERR_NVML

    cq_nvml_init = cq_nvml_energy_mj = cq_nvml_power_mw = cq_nvml_sm_clock_mhz = _nvml_absent
    cq_nvml_throttle_reasons = cq_nvml_supported_sm_clocks = _nvml_absent
    cq_nvml_lock_sm_clock = cq_nvml_reset_sm_clock = _nvml_absent


class FakeNvmlLib(FakeLib):
    """FakeLib plus a simulated NVML device: a lockable SM clock and an
    energy counter integrating P(f) = static + dynamic * (f / f_max)^3 over
    wall time (for the SYnergy sweep logic on CPU)."""

    CLOCKS = (1965, 1800, 1500, 1200, 990, 600)

    def __init__(self, *a, allow_lock=True, tick_s=0.0, **kw):
        super().__init__(*a, **kw)
        import time as _t
        self._t = _t
        self.mhz = max(self.CLOCKS)
        self.allow_lock = allow_lock
        self.tick_s = tick_s  # > 0: the counter publishes in steps, like NVML's
        self._mj = 0.0
        self._last = self._tick = _t.perf_counter()
        self._published = 0

    def _power_w(self):
        return 200.0 + 800.0 * (self.mhz / max(self.CLOCKS)) ** 3

    def _advance(self):
        now = self._t.perf_counter()
        self._mj += self._power_w() * (now - self._last) * 1000.0
        self._last = now

    def cq_nvml_init(self):
        return 0

    def cq_nvml_energy_mj(self, d, p):
        self._advance()
        if self.tick_s <= 0 or self._last - self._tick >= self.tick_s:
            self._published, self._tick = int(self._mj), self._last
        _obj(p).value = self._published
        return 0

    def cq_nvml_power_mw(self, d, p):
        _obj(p).value = int(self._power_w() * 1000)
        return 0

    def cq_nvml_sm_clock_mhz(self, d, cur, mx):
        _obj(cur).value, _obj(mx).value = self.mhz, max(self.CLOCKS)
        return 0

    def cq_nvml_throttle_reasons(self, d, p):
        _obj(p).value = 0
        return 0

    def cq_nvml_supported_sm_clocks(self, d, buf, n):
        arr = _obj(buf)
        for i, c in enumerate(self.CLOCKS):
            arr[i] = c
        _obj(n).value = len(self.CLOCKS)
        return 0

    def cq_nvml_lock_sm_clock(self, d, mhz):
        if not self.allow_lock:
            self.err = b"clock locking disabled (CQ_ALLOW_CLOCK_LOCK)"
            return N.CQ_ERR_PERMISSION
        self._advance()
        self.mhz = int(_val(mhz))
        return 0

    def cq_nvml_reset_sm_clock(self, d):
        self._advance()
        self.mhz = max(self.CLOCKS)
        return 0


class LocalTransport:
    """Single process: NCCL ops must never be issued."""

    def exchange(self, ops, lib):
        if ops:
            raise AssertionError("NCCL op issued in a single-process run")

    def allgather(self, lib, send, recv, n):
        raise AssertionError("NCCL all-gather issued in a single-process run")

    def bcast(self, lib, buf, n, root):
        raise AssertionError("NCCL broadcast issued in a single-process run")


class GlooTransport:
    """NCCL group semantics over torch.distributed (gloo): all sends and
    receives of a group are posted together, so matching across ranks must
    be consistent or the test deadlocks / mismatches sizes."""

    def exchange(self, ops, lib):
        import torch
        import torch.distributed as dist
        reqs = []
        recvs = []
        for op, addr, n, peer in ops:
            if op == "send":
                t = torch.from_numpy(lib._mem(addr, n).copy())
                reqs.append(dist.isend(t, peer))
            else:
                t = torch.empty(n, dtype=torch.uint8)
                reqs.append(dist.irecv(t, peer))
                recvs.append((addr, n, t))
        for r in reqs:
            r.wait()
        for addr, n, t in recvs:
            lib._mem(addr, n)[:] = t.numpy()
        lib.launches.append(("group", len(ops)))

    def allgather(self, lib, send, recv, n):
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(), dist.get_rank()
        assert send == recv + rank * n, "all-gather must be in place (rank r's chunk at recv + r * n)"
        t = torch.from_numpy(lib._mem(send, n).copy())
        out = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(out, t)
        for r, o in enumerate(out):
            lib._mem(recv + r * n, n)[:] = o.numpy()

    def bcast(self, lib, buf, n, root):
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(lib._mem(buf, n).copy())
        dist.broadcast(t, root)
        lib._mem(buf, n)[:] = t.numpy()


def _graph_api(cls):
    """Graph capture in the double: record the issued calls and re-issue
    them on launch (enough to exercise Session.capture/replay on CPU)."""
    def begin(self, d):
        self.capturing = []
        return 0

    def end(self, d, p):
        self.graphs = getattr(self, "graphs", [])
        self.graphs.append(self.capturing)
        self.capturing = None
        _obj(p).value = len(self.graphs)
        return 0

    def launch(self, g, d):
        for name, args in self.graphs[_val(g) - 1]:
            getattr(cls, name)(self, *args)
        return 0

    def destroy(self, g):
        return 0
    cls.cq_graph_begin, cls.cq_graph_end = begin, end
    cls.cq_graph_launch, cls.cq_graph_destroy = launch, destroy
    # wrap kernel entry points so they are recorded while capturing
    for name in ("cq_saxpy", "cq_wave5", "cq_wave5_fused", "cq_expr_eval", "cq_fill", "cq_copy_box", "cq_pack_box",
                 "cq_unpack_box", "cq_nbody_kick", "cq_nbody_drift", "cq_sgemm", "cq_nbody_kick_partial",
                 "cq_nbody_kick_finalize"):
        fn = getattr(cls, name)

        def wrapped(self, *args, _fn=fn, _name=name):
            if getattr(self, "capturing", None) is not None:
                self.capturing.append((_name, _copy_args(args)))
                return 0
            return _fn(self, *args)
        setattr(cls, name, wrapped)
    return cls


def _copy_args(args):
    out = []
    for a in args:
        o = _obj(a)
        if isinstance(o, ctypes.Structure):
            c = type(o)()
            ctypes.pointer(c)[0] = o
            out.append(c)
        else:
            out.append(_val(a))
    return out


_graph_api(FakeLib)
