"""ctypes binding of libdg_b200.so (include/distgrid_b200.h) — the Python face of the
drop-in boundary, used by tests/, bench.py and __graft_entry__.

Mirrors the reference's DistributedRun surface (worker.hpp:182-226):
    ctx.train_step(origin, dir, color_gt, image_id, step) -> StepStats   (training_step)
    ctx.render(origin, dir, appearance)                     -> (rgb, T, depth) (evaluate_rays)
plus state injection/extraction (params, Adam moments, occupancy) for parity.

There is no fallback: if the CUDA library is missing this module raises on load.
"""
import ctypes as C
import os
import re

import numpy as np

from . import abi
from .abi import (DG_MAX_SEGMENTS, DG_MEM_DEVICE, DG_MEM_HOST, ArrayDesc, ItemView, Merged,
                  RayBatch, RunConfig, StageTimes, StepStats)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DG_LIB") or os.path.join(HERE, "libdg_b200.so")  # DG_LIB: A/B builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "distgrid_b200.h")

P = C.c_void_p


class DGError(RuntimeError):
    """Maps dg_status codes onto the reference's exception classes by name."""

    def __init__(self, code, msg):
        self.code = code
        self.status = abi.STATUS_NAMES.get(code, str(code))
        super().__init__(f"{self.status}: {msg}")


_lib = None


def header_functions():
    """Names of every dg_* function declared in include/distgrid_b200.h."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(", text)) - {"dg_alltoallv_fn"})


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.dg_last_error.restype = C.c_char_p
        L.dg_lr_at.restype = C.c_double
        L.dg_lr_at.argtypes = [C.POINTER(RunConfig), C.c_uint64]
        L.dg_default_config.argtypes = [C.POINTER(RunConfig)]
        L.dg_ctx_create.argtypes = [C.POINTER(RunConfig), C.c_int, C.c_int, C.c_int, C.POINTER(P)]
        L.dg_ctx_destroy.argtypes = [P]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise DGError(rc, lib().dg_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(P)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _c32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Context:
    """One dg_ctx: the partitions of `rank` on `device` (partition p lives on rank p % world)."""

    def __init__(self, cfg, device=-1, rank=0, world=1):
        L = lib()
        self.cfg = cfg.copy()
        self.h = P()
        _check(L.dg_ctx_create(C.byref(self.cfg), device, rank, world, C.byref(self.h)))
        self.rank, self.world = rank, world
        nt, nl = C.c_uint32(), C.c_uint32()
        _check(L.dg_partition_count(self.h, C.byref(nt), C.byref(nl)))
        self.P = nt.value
        self.local = [p for p in range(self.P) if p % world == rank]
        self._cb = None

    def close(self):
        if getattr(self, "h", None):
            lib().dg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- geometry / layout ----
    @property
    def march_step(self):
        v = C.c_double()
        _check(lib().dg_march_step(self.h, C.byref(v)))
        return v.value

    def param_count(self, g):
        n = C.c_uint64()
        _check(lib().dg_param_count(self.h, C.c_uint32(g), C.byref(n)))
        return n.value

    def param_layout(self, g):
        arr = (ArrayDesc * 64)()
        n = C.c_uint32()
        _check(lib().dg_param_layout(self.h, C.c_uint32(g), arr, 64, C.byref(n)))
        return [dict(offset=a.offset, size=a.size, cascade=a.cascade, kind=a.kind, index=a.index)
                for a in arr[:n.value]]

    def grid_levels(self, g, cascade):
        L = self.cfg.grid_levels
        shapes = np.zeros((L, 3), dtype=np.uint32)
        modes = np.zeros(L, dtype=np.uint32)
        rows = np.zeros(L, dtype=np.uint64)
        _check(lib().dg_grid_levels(self.h, C.c_uint32(g), C.c_uint32(cascade), _p(shapes),
                                    _p(modes), _p(rows)))
        return shapes, modes, rows

    def occupancy_shape(self, g, cascade):
        s = (C.c_uint32 * 3)()
        _check(lib().dg_occupancy_shape(self.h, C.c_uint32(g), C.c_uint32(cascade), s))
        return tuple(s)

    # ---- state ----
    def set_params(self, g, p):
        p = _c32(p)
        assert p.size == self.param_count(g)
        _check(lib().dg_set_params(self.h, C.c_uint32(g), _p(p)))

    def get_params(self, g):
        out = np.zeros(self.param_count(g), dtype=np.float32)
        _check(lib().dg_get_params(self.h, C.c_uint32(g), _p(out)))
        return out

    def get_grads(self, g):
        out = np.zeros(self.param_count(g), dtype=np.float32)
        _check(lib().dg_get_grads(self.h, C.c_uint32(g), _p(out)))
        return out

    def zero_grads(self):
        _check(lib().dg_zero_grads(self.h))

    def set_adam(self, g, m, v, t):
        m, v = _c32(m), _c32(v)
        _check(lib().dg_set_adam(self.h, C.c_uint32(g), _p(m), _p(v), C.c_uint64(t)))

    def get_adam(self, g):
        n = self.param_count(g)
        m = np.zeros(n, dtype=np.float32)
        v = np.zeros(n, dtype=np.float32)
        t = C.c_uint64()
        _check(lib().dg_get_adam(self.h, C.c_uint32(g), _p(m), _p(v), C.byref(t)))
        return m, v, t.value

    def set_step(self, s):
        _check(lib().dg_set_step(self.h, C.c_uint64(s)))

    def get_step(self):
        v = C.c_uint64()
        _check(lib().dg_get_step(self.h, C.byref(v)))
        return v.value

    def snapshot(self, restore=False):
        """dg_state_snapshot: take (restore=False) or restore the device-side training state."""
        _check(lib().dg_state_snapshot(self.h, 1 if restore else 0))

    def init_reference(self, g):
        _check(lib().dg_init_params_reference(self.h, C.c_uint32(g)))

    def init_fast(self, g, seed=1):
        _check(lib().dg_init_params_fast(self.h, C.c_uint32(g), C.c_uint64(seed)))

    def set_occupancy(self, g, cascade, bits):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        _check(lib().dg_set_occupancy(self.h, C.c_uint32(g), C.c_uint32(cascade), _p(bits)))

    def get_occupancy(self, g, cascade):
        s = self.occupancy_shape(g, cascade)
        bits = np.zeros(s[0] * s[1] * s[2], dtype=np.uint8)
        _check(lib().dg_get_occupancy(self.h, C.c_uint32(g), C.c_uint32(cascade), _p(bits)))
        return bits

    def save_checkpoint(self, g, config_hash, path):
        """The reference's .dgcw file for partition g (checkpoint.cpp:241-258)."""
        _check(lib().dg_save_checkpoint(self.h, C.c_uint32(g), C.c_uint64(config_hash), str(path).encode()))

    def load_checkpoint(self, g, path):
        """Load a .dgcw (reference- or GPU-written) into partition g; returns its config hash."""
        h = C.c_uint64()
        _check(lib().dg_load_checkpoint(self.h, C.c_uint32(g), str(path).encode(), C.byref(h)))
        return h.value

    def occupancy_density(self, g, cascade):
        sh = self.occupancy_shape(g, cascade)
        den = np.zeros(int(np.prod(sh)), np.float32)
        thr = C.c_double()
        _check(lib().dg_get_occupancy_density(self.h, C.c_uint32(g), C.c_uint32(cascade), _p(den), C.byref(thr)))
        return den, thr.value

    def set_appearance(self, rows, ids=None):
        rows = _c32(np.atleast_2d(rows))
        ids = np.arange(rows.shape[0], dtype=np.uint32) if ids is None else \
            np.ascontiguousarray(ids, dtype=np.uint32)
        _check(lib().dg_set_appearance(self.h, _p(ids), _p(rows), C.c_uint32(rows.shape[0])))

    # ---- composed path ----
    def _batch(self, origin, dir, color_gt=None, image_id=None, first_ray_id=0):
        b = RayBatch()
        self._keep = [_c64(origin), _c64(dir),
                      None if color_gt is None else _c32(color_gt),
                      None if image_id is None else np.ascontiguousarray(image_id, dtype=np.uint32)]
        o, d, gt, img = self._keep
        b.origin, b.dir, b.color_gt, b.image_id = _p(o), _p(d), _p(gt), _p(img)
        b.n = len(o)
        b.first_ray_id = first_ray_id
        b.mem = DG_MEM_HOST
        return b

    def train_step(self, origin, dir, color_gt, image_id=None, step=0, first_ray_id=0):
        b = self._batch(origin, dir, color_gt, image_id, first_ray_id)
        st = StepStats()
        _check(lib().dg_train_step(self.h, C.byref(b), C.c_uint64(step), C.byref(st)))
        return {k: getattr(st, k) for k, _ in StepStats._fields_}

    def train_step_raw(self, batch, step, stats):
        """Zero-copy variant for pre-built RayBatch structs (device or pinned host)."""
        return lib().dg_train_step(self.h, C.byref(batch), C.c_uint64(step), C.byref(stats))

    def render_image(self, camera, appearance):
        """evaluate_image (worker.cpp:836-880) for a camera dict: rgb, T, depth, attribution."""
        from .abi import cameras
        cam = cameras([camera])
        n = camera["width"] * camera["height"]
        rgb, T, depth = np.zeros((n, 3), np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32)
        attr = np.zeros((n, 3), np.float32)
        m = Merged()
        m.rgb, m.transmittance, m.depth, m.attribution, m.mem = _p(rgb), _p(T), _p(depth), _p(attr), DG_MEM_HOST
        app = _c32(appearance)
        _check(lib().dg_render_image(self.h, cam, _p(app), C.byref(m)))
        return rgb, T, depth, attr

    def render(self, origin, dir, appearance, first_ray_id=0, attribution=False):
        b = self._batch(origin, dir, None, None, first_ray_id)
        n = b.n
        rgb = np.zeros((n, 3), dtype=np.float32)
        T = np.zeros(n, dtype=np.float32)
        depth = np.zeros(n, dtype=np.float32)
        attr = np.zeros((n, 3), dtype=np.float32) if attribution else None
        m = Merged()
        m.rgb, m.transmittance, m.depth, m.mem = _p(rgb), _p(T), _p(depth), DG_MEM_HOST
        m.attribution = _p(attr)
        app = _c32(appearance)
        _check(lib().dg_render(self.h, C.byref(b), _p(app), C.byref(m)))
        return (rgb, T, depth, attr) if attribution else (rgb, T, depth)

    def render_raw(self, batch, app, merged):
        return lib().dg_render(self.h, C.byref(batch), _p(app), C.byref(merged))

    # ---- comms ----
    def comm_init_nccl(self, uid_bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid_bytes))
        _check(lib().dg_comm_init_nccl(self.h, buf))

    def set_comm_timeout(self, ms):
        """Worker::Setup::recv_timeout (worker.hpp:82): DG_ETIMEOUT after `ms` without peers."""
        _check(lib().dg_set_comm_timeout(self.h, C.c_uint64(int(ms))))

    def comm_init_host(self, fn):
        """fn(send: bytes-like per peer list, recv_sizes) -> list of received bytes (rank order)."""
        proto = C.CFUNCTYPE(C.c_int, P, P, C.POINTER(C.c_uint64), P, C.POINTER(C.c_uint64))

        def cb(user, send, send_bytes, recv, recv_bytes):
            try:
                W = self.world
                sb = [send_bytes[i] for i in range(W)]
                rb = [recv_bytes[i] for i in range(W)]
                total = sum(sb)
                blob = C.string_at(send, total) if total else b""
                blocks, off = [], 0
                for s in sb:
                    blocks.append(blob[off:off + s])
                    off += s
                got = fn(blocks, rb)
                off = 0
                for r in range(W):
                    assert len(got[r]) == rb[r], (r, len(got[r]), rb[r])
                    if rb[r]:
                        C.memmove(recv + off, got[r], rb[r])
                    off += rb[r]
                return 0
            except Exception as e:  # surfaces as DG_ETIMEOUT
                import traceback
                traceback.print_exc()
                return 1

        self._cb = proto(cb)
        _check(lib().dg_comm_init_host(self.h, self._cb, None))

    def comm_init_peer(self, allgather):
        """Peer-memory backend (dg_comm_init_peer): allgather(bytes) -> list of every rank's
        bytes (rank order), e.g. torch.distributed.all_gather_object over gloo."""
        proto = C.CFUNCTYPE(C.c_int, P, P, C.c_uint64, P)

        def cb(user, send, nbytes, recv):
            try:
                got = allgather(C.string_at(send, nbytes) if nbytes else b"")
                off = 0
                for blob in got:
                    assert len(blob) == nbytes, (len(blob), nbytes)
                    if nbytes:
                        C.memmove(recv + off, blob, nbytes)
                    off += nbytes
                return 0
            except Exception:  # surfaces as DG_ETIMEOUT
                import traceback
                traceback.print_exc()
                return 1

        self._cb = proto(cb)
        _check(lib().dg_comm_init_peer(self.h, self._cb, None))

    # ---- stage entry points ----
    def segment_rays(self, origin, dir):
        o, d = _c64(origin), _c64(dir)
        n = len(o)
        nseg = np.zeros(n, dtype=np.uint8)
        region = np.zeros((n, DG_MAX_SEGMENTS), dtype=np.uint16)
        te = np.zeros((n, DG_MAX_SEGMENTS))
        tx = np.zeros((n, DG_MAX_SEGMENTS))
        _check(lib().dg_segment_rays(self.h, _p(o), _p(d), C.c_uint64(n), _p(nseg), _p(region),
                                     _p(te), _p(tx), DG_MEM_HOST))
        return nseg, region, te, tx

    def cascade_march(self, g, origin, dir, t0, t1, ray_id, jitter, batch_id):
        o, d, a, b = _c64(origin), _c64(dir), _c64(t0), _c64(t1)
        rid = np.ascontiguousarray(ray_id, dtype=np.uint64)
        n = len(o)
        counts = np.zeros(n, dtype=np.uint32)
        args = (self.h, C.c_uint32(g), _p(o), _p(d), _p(a), _p(b), _p(rid), C.c_uint64(n),
                C.c_int32(int(jitter)), C.c_uint64(batch_id))
        _check(lib().dg_cascade_march(*args, _p(counts), None, None, None, None, DG_MEM_HOST))
        off = np.zeros(n, dtype=np.uint64)
        off[1:] = np.cumsum(counts.astype(np.uint64))[:-1]
        tot = int(counts.sum())
        t = np.zeros(max(tot, 1))
        delta = np.zeros(max(tot, 1))
        casc = np.zeros(max(tot, 1), dtype=np.uint8)
        _check(lib().dg_cascade_march(*args, _p(counts), _p(off), _p(t), _p(delta), _p(casc),
                                      DG_MEM_HOST))
        return counts, t[:tot], delta[:tot], casc[:tot]

    def encode(self, g, cascade, points, with_rows=True):
        pts = _c64(points)
        n = len(pts)
        Lf = self.cfg.grid_levels * 2
        feats = np.zeros((n, Lf), dtype=np.float32)
        rows = np.zeros((n, self.cfg.grid_levels, 8), dtype=np.uint32) if with_rows else None
        _check(lib().dg_encode(self.h, C.c_uint32(g), C.c_uint32(cascade), _p(pts), C.c_uint64(n),
                               _p(feats), _p(rows), DG_MEM_HOST))
        return feats, rows

    def encode_backward(self, g, cascade, points, upstream):
        pts, up = _c64(points), _c32(upstream)
        _check(lib().dg_encode_backward(self.h, C.c_uint32(g), C.c_uint32(cascade), _p(pts),
                                        _p(up), C.c_uint64(len(pts)), DG_MEM_HOST))

    def field_forward(self, g, cascade, points, dirs, app):
        pts, dd, aa = _c64(points), _c32(dirs), _c32(app)
        n = len(pts)
        sigma = np.zeros(n, dtype=np.float32)
        rgb = np.zeros((n, 3), dtype=np.float32)
        _check(lib().dg_field_forward(self.h, C.c_uint32(g), C.c_uint32(cascade), _p(pts), _p(dd),
                                      _p(aa), C.c_uint64(n), _p(sigma), _p(rgb), DG_MEM_HOST))
        return sigma, rgb

    def field_backward(self, g, cascade, points, dirs, app, dsigma, drgb):
        pts, dd, aa, ds, dr = _c64(points), _c32(dirs), _c32(app), _c32(dsigma), _c32(drgb)
        _check(lib().dg_field_backward(self.h, C.c_uint32(g), C.c_uint32(cascade), _p(pts), _p(dd),
                                       _p(aa), _p(ds), _p(dr), C.c_uint64(len(pts)), DG_MEM_HOST))

    def adam_step(self, lr):
        _check(lib().dg_adam_step(self.h, C.c_double(lr)))

    # ---- compositing stages (render.hpp / train.hpp, batched; host arrays) ----
    def local_render(self, t, delta, sigma, rgb, seg_off, ray_t0=None, ray_t1=None):
        """local_render per segment (+ accumulate_distortion_stats when the ray span is given).
        Returns rgb [n_seg, 3], T, depth_sum (and distortion stats [n_seg, 3])."""
        off = np.ascontiguousarray(seg_off, dtype=np.uint64)
        ns = len(off) - 1
        out_rgb = np.zeros((ns, 3), np.float32)
        out_T = np.zeros(ns, np.float32)
        out_d = np.zeros(ns, np.float32)
        dist = None if ray_t0 is None else np.zeros((ns, 3))
        _check(lib().dg_local_render(self.h, _p(_c64(t)), _p(_c64(delta)), _p(_c32(sigma)), _p(_c32(rgb)),
                                     _p(off), C.c_uint64(ns), _p(None if ray_t0 is None else _c64(ray_t0)),
                                     _p(None if ray_t1 is None else _c64(ray_t1)), _p(out_rgb), _p(out_T),
                                     _p(out_d), _p(dist), DG_MEM_HOST))
        return (out_rgb, out_T, out_d) if dist is None else (out_rgb, out_T, out_d, dist)

    def local_render_backward(self, t, delta, sigma, rgb, seg_off, d_rgb, d_T, weight_up=None):
        off = np.ascontiguousarray(seg_off, dtype=np.uint64)
        ns, n = len(off) - 1, int(off[-1])
        sg = np.zeros(n, np.float32)
        cg = np.zeros((n, 3), np.float32)
        _check(lib().dg_local_render_backward(self.h, _p(_c64(t)), _p(_c64(delta)), _p(_c32(sigma)),
                                              _p(_c32(rgb)), _p(off), C.c_uint64(ns), _p(_c32(d_rgb)),
                                              _p(_c32(d_T)), _p(None if weight_up is None else _c32(weight_up)),
                                              _p(sg), _p(cg), DG_MEM_HOST))
        return sg, cg

    def merge_forward(self, seg_rgb, seg_T, seg_depth, ray_off):
        off = np.ascontiguousarray(ray_off, dtype=np.uint64)
        nr = len(off) - 1
        rgb = np.zeros((nr, 3), np.float32)
        T = np.zeros(nr, np.float32)
        depth = np.zeros(nr, np.float32)
        _check(lib().dg_merge_forward(self.h, _p(_c32(seg_rgb)), _p(_c32(seg_T)), _p(_c32(seg_depth)), _p(off),
                                      C.c_uint64(nr), _p(rgb), _p(T), _p(depth), DG_MEM_HOST))
        return rgb, T, depth

    def merge_backward(self, seg_rgb, seg_T, ray_off, d_rgb, d_T):
        off = np.ascontiguousarray(ray_off, dtype=np.uint64)
        nr, ns = len(off) - 1, int(off[-1])
        g_rgb = np.zeros((ns, 3), np.float32)
        g_T = np.zeros(ns, np.float32)
        _check(lib().dg_merge_backward(self.h, _p(_c32(seg_rgb)), _p(_c32(seg_T)), _p(off), C.c_uint64(nr),
                                       _p(_c32(d_rgb)), _p(_c32(d_T)), _p(g_rgb), _p(g_T), DG_MEM_HOST))
        return g_rgb, g_T

    def ray_losses(self, rgb, gt, T, eps=1e-6):
        n = len(T)
        lr, lt = np.zeros(n), np.zeros(n)
        dr, dt = np.zeros((n, 3), np.float32), np.zeros(n, np.float32)
        _check(lib().dg_ray_losses(self.h, _p(_c32(rgb)), _p(_c32(gt)), _p(_c32(T)), C.c_uint64(n),
                                   C.c_double(eps), _p(lr), _p(lt), _p(dr), _p(dt), DG_MEM_HOST))
        return lr, lt, dr, dt

    def distortion_loss(self, w, s, ds, seg_off):
        off = np.ascontiguousarray(seg_off, dtype=np.uint64)
        ns, n = len(off) - 1, int(off[-1])
        loss, grads = np.zeros(ns), np.zeros(n)
        _check(lib().dg_distortion_loss(self.h, _p(_c64(w)), _p(_c64(s)), _p(_c64(ds)), _p(off), C.c_uint64(ns),
                                        _p(loss), _p(grads), DG_MEM_HOST))
        return loss, grads

    # ---- introspection ----
    def last_items(self, g):
        v = ItemView()
        _check(lib().dg_last_items(self.h, C.c_uint32(g), C.byref(v)))
        return v.n_items, v.n_fine, v.n_coarse

    def last_item_data(self, g):
        n, _, _ = self.last_items(g)
        rid = np.zeros(n, dtype=np.uint64)
        order = np.zeros(n, dtype=np.uint8)
        te = np.zeros(n)
        tx = np.zeros(n)
        ns = np.zeros(n, dtype=np.uint32)
        _check(lib().dg_last_item_data(self.h, C.c_uint32(g), _p(rid), _p(order), _p(te), _p(tx),
                                       _p(ns)))
        return rid, order, te, tx, ns

    def last_samples(self, g):
        _, nf, nc = self.last_items(g)
        tot = nf + nc
        t = np.zeros(max(tot, 1))
        d = np.zeros(max(tot, 1))
        c = np.zeros(max(tot, 1), dtype=np.uint8)
        _check(lib().dg_last_samples(self.h, C.c_uint32(g), _p(t), _p(d), _p(c)))
        return t[:tot], d[:tot], c[:tot]

    def last_sample_data(self, g, masks=False):
        """(pos [n,3], features [n,2L], field_out [n,4], upstream [n,4], d_features [n,2L]
        [, masks [n,7]]) of the last training step's samples of partition g, in last_samples
        order."""
        _, nf, nc = self.last_items(g)
        n, L2 = nf + nc, 2 * self.cfg.grid_levels
        pos = np.zeros((max(n, 1), 3))
        x = np.zeros((max(n, 1), L2), dtype=np.float32)
        out = np.zeros((max(n, 1), 4), dtype=np.float32)
        up = np.zeros((max(n, 1), 4), dtype=np.float32)
        dx = np.zeros((max(n, 1), L2), dtype=np.float32)
        mk = np.zeros((max(n, 1), 7), dtype=np.uint32) if masks else None
        _check(lib().dg_last_sample_data(self.h, C.c_uint32(g), _p(pos), _p(x), _p(out), _p(up), _p(dx),
                                         _p(mk)))
        res = (pos[:n], x[:n], out[:n], up[:n], dx[:n])
        return res + (mk[:n],) if masks else res

    def last_masks(self, g):
        """The tcgen05 forward's ReLU / clip mask words [n, 7] of the last training step's samples
        of partition g (last_samples order); raises DG_EINVAL on the FFMA path."""
        _, nf, nc = self.last_items(g)
        n = nf + nc
        mk = np.zeros((max(n, 1), 7), dtype=np.uint32)
        _check(lib().dg_last_sample_data(self.h, C.c_uint32(g), None, None, None, None, None, _p(mk)))
        return mk[:n]

    def last_partials(self, g):
        n, _, _ = self.last_items(g)
        rgb = np.zeros((n, 3), dtype=np.float32)
        T = np.zeros(n, dtype=np.float32)
        _check(lib().dg_last_partials(self.h, C.c_uint32(g), _p(rgb), _p(T)))
        return rgb, T

    def stream(self):
        v = C.c_void_p()
        _check(lib().dg_get_stream(self.h, C.byref(v)))
        return v.value

    def set_stream(self, stream_ptr):
        """Run later calls on the caller's cudaStream_t (an int handle, e.g.
        torch.cuda.Stream().cuda_stream); None returns to the context's own stream."""
        _check(lib().dg_set_stream(self.h, C.c_void_p(stream_ptr)))

    def kernel_launches(self):
        v = C.c_uint64()
        _check(lib().dg_kernel_launches(self.h, C.byref(v)))
        return v.value

    def enable_stage_timing(self, on=True):
        _check(lib().dg_enable_stage_timing(self.h, int(on)))

    def stage_times(self):
        t = StageTimes()
        _check(lib().dg_last_stage_times(self.h, C.byref(t)))
        return t.as_dict()

    def synchronize(self):
        _check(lib().dg_synchronize(self.h))

    def fence(self):
        """Order the context stream after the last step's (side-stream) Adam update."""
        _check(lib().dg_fence(self.h))


def lr_at(cfg, step):
    return lib().dg_lr_at(C.byref(cfg), C.c_uint64(step))


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    _check(lib().dg_comm_unique_id(buf))
    return bytes(buf)


# ---- exchange planning (host only; include/distgrid_b200.h dg_plan_*) ----
def plan_dispatch(rank, world, P, send_cnt, cnt_recv):
    """Exchange-1 layouts: (send_bytes[W], recv_bytes[W], item_off[nl+1], block_src, block_dst)."""
    nl = len([p for p in range(P) if p % world == rank])
    sc = np.ascontiguousarray(send_cnt, dtype=np.uint64)
    cr = np.ascontiguousarray(cnt_recv, dtype=np.uint64).reshape(-1)
    sb = np.zeros(world, np.uint64)
    rb = np.zeros(world, np.uint64)
    io = np.zeros(nl + 1, np.uint32)
    bs = np.zeros(max(1, world * nl), np.uint64)
    bd = np.zeros(max(1, world * nl), np.uint64)
    _check(lib().dg_plan_dispatch(C.c_int(rank), C.c_int(world), C.c_uint32(P), _p(sc), _p(cr), _p(sb),
                                  _p(rb), _p(io), _p(bs), _p(bd)))
    return sb, rb, io, bs[:world * nl], bd[:world * nl]


def plan_partials(rank, world, P, pair_cnt):
    """Exchange-2 layouts: (send_off[P,P], recv_off[P,P], send_bytes[W], recv_bytes[W])."""
    pc = np.ascontiguousarray(pair_cnt, dtype=np.uint32).reshape(-1)
    so = np.zeros(P * P, np.uint64)
    ro = np.zeros(P * P, np.uint64)
    sb = np.zeros(world, np.uint64)
    rb = np.zeros(world, np.uint64)
    _check(lib().dg_plan_partials(C.c_int(rank), C.c_int(world), C.c_uint32(P), _p(pc), _p(so), _p(ro),
                                  _p(sb), _p(rb)))
    return so.reshape(P, P), ro.reshape(P, P), sb, rb


# ---- ray cache / pixel-ray batch feed (dg_ray_cache_*) ----
class RayCache:
    """Device-resident RayCache (train.cpp:117-159): images + poses uploaded once; refresh()
    builds rays on the GPU, draw() returns a device RayBatch that train_step_raw consumes."""

    def __init__(self, poses, images, capacity, seed, device=-1):
        from .abi import cameras
        self._cams = cameras(poses)
        self._imgs = [np.ascontiguousarray(im, dtype=np.uint8) for im in images]
        ptrs = (C.c_void_p * len(self._imgs))(*[im.ctypes.data for im in self._imgs])
        self.h = P()
        _check(lib().dg_ray_cache_create(C.c_int(device), self._cams, ptrs, C.c_uint32(len(self._imgs)),
                                         C.c_uint64(capacity), C.c_uint64(seed), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().dg_ray_cache_destroy(self.h)
            self.h = None

    def size(self):
        n, cap = C.c_uint64(), C.c_uint64()
        _check(lib().dg_ray_cache_size(self.h, C.byref(n), C.byref(cap)))
        return n.value

    def refresh(self, count):
        _check(lib().dg_ray_cache_refresh(self.h, C.c_uint64(count)))

    def draw(self, n):
        b = RayBatch()
        _check(lib().dg_ray_cache_draw(self.h, C.c_uint64(n), C.byref(b)))
        return b

    def snapshot(self):
        n = self.size()
        o, d = np.zeros((n, 3)), np.zeros((n, 3))
        gt = np.zeros((n, 3), np.float32)
        img = np.zeros(n, np.uint32)
        pix = np.zeros(n, np.uint64)
        _check(lib().dg_ray_cache_snapshot(self.h, _p(o), _p(d), _p(gt), _p(img), _p(pix)))
        return o, d, gt, img, pix
