"""TEST INFRASTRUCTURE: ctypes bindings of the oracle libraries.

  Oracle      — oracle/build/liboracle.so, the C restatement (dg_oracle.c).
  Reference   — oracle/_ref/libdistgrid_ref.so, the unmodified reference library built from
                /root/reference sources + ref_harness.cpp.  Present only where it was built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs import
this module.  The product path (paper_2405_04416_b200) never does.
"""
import ctypes as C
import os

import numpy as np

from paper_2405_04416_b200.abi import DG_MAX_SEGMENTS, RunConfig

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdistgrid_ref.so")

P = C.c_void_p
U8 = np.uint8


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def build_oracle():
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        lib = C.CDLL(ORACLE_SO)
        lib.or_run_create.restype = P
        lib.or_run_create.argtypes = [C.POINTER(RunConfig), C.c_uint32, P]
        lib.or_run_destroy.argtypes = [P]
        for name in ("or_run_params", "or_run_grads", "or_run_adam_m", "or_run_adam_v",
                     "or_run_occ_density", "or_run_abs_grads"):
            getattr(lib, name).restype = C.POINTER(C.c_double)
        lib.or_run_params.argtypes = [P, C.c_uint32]
        lib.or_run_grads.argtypes = [P, C.c_uint32]
        lib.or_run_abs_grads.argtypes = [P, C.c_uint32]
        lib.or_run_adam_m.argtypes = [P, C.c_uint32]
        lib.or_run_adam_v.argtypes = [P, C.c_uint32]
        lib.or_run_occ_density.argtypes = [P, C.c_uint32, C.c_uint32]
        lib.or_run_adam_t.restype = C.POINTER(C.c_uint64)
        lib.or_run_adam_t.argtypes = [P, C.c_uint32]
        lib.or_run_worker_step.restype = C.POINTER(C.c_uint64)
        lib.or_run_worker_step.argtypes = [P, C.c_uint32]
        lib.or_run_occ_bits.restype = C.POINTER(C.c_uint8)
        lib.or_run_occ_bits.argtypes = [P, C.c_uint32, C.c_uint32]
        lib.or_run_set_occupancy.argtypes = [P, C.c_uint32, C.c_uint32, P]
        lib.or_run_train_step.argtypes = [P, P, P, P, P, C.c_uint64, C.c_uint64, P]
        lib.or_run_sample_log.argtypes = [P, C.c_int32, P, C.c_uint64]
        lib.or_run_mask_override.argtypes = [P, C.c_uint32, P, C.c_uint64]
        lib.or_run_override_stats.argtypes = [P, P, P]
        lib.or_run_sample_log_count.argtypes = [P]
        lib.or_run_sample_log_count.restype = C.c_uint64
        lib.or_run_eval_rays.argtypes = [P, P, P, C.c_uint64, P, P, P, P]
        lib.or_last_error.restype = C.c_char_p
        lib.or_run_model.restype = P
        lib.or_segment_ray.argtypes = [P, P, P, P, P, P]
        lib.or_counter_uniform.restype = C.c_double
        lib.or_counter_uniform.argtypes = [C.c_uint64] * 4
        lib.or_counter_hash.restype = C.c_uint64
        lib.or_counter_hash.argtypes = [C.c_uint64] * 4
        lib.or_lr_at.restype = C.c_double
        lib.or_lr_at.argtypes = [C.POINTER(RunConfig), C.c_uint64]
        lib.or_level_resolution.restype = C.c_uint32
        lib.or_level_resolution.argtypes = [C.c_uint32] * 4
        _oracle = lib
    return _oracle


def ref_available():
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError("reference build missing: " + REF_SO)
        lib = C.CDLL(REF_SO)
        lib.refh_create.restype = P
        lib.refh_create.argtypes = [C.POINTER(RunConfig), C.c_uint32, P]
        lib.refh_destroy.argtypes = [P]
        lib.refh_param_count.restype = C.c_uint64
        lib.refh_param_count.argtypes = [P, C.c_uint32]
        lib.refh_get_params.argtypes = [P, C.c_uint32, P]
        lib.refh_set_params.argtypes = [P, C.c_uint32, P]
        lib.refh_get_adam.argtypes = [P, C.c_uint32, P, P, P, P]
        lib.refh_set_adam.argtypes = [P, C.c_uint32, P, P, C.c_uint64, C.c_uint64]
        lib.refh_set_occupancy.argtypes = [P, C.c_uint32, C.c_uint32, P]
        lib.refh_get_occupancy.argtypes = [P, C.c_uint32, C.c_uint32, P, P]
        lib.refh_train_step.argtypes = [P, P, P, P, P, C.c_uint64, C.c_uint64, P]
        lib.refh_eval_rays.argtypes = [P, P, P, C.c_uint64, P, P, P, P]
        lib.refh_segment_rays.argtypes = [C.POINTER(RunConfig), P, P, C.c_uint64, P, P, P, P]
        lib.refh_cascade_march.argtypes = [P, C.c_uint32, P, P, P, P, P, C.c_uint64, C.c_int,
                                           C.c_uint64, P, P, P, P, C.c_uint64]
        lib.refh_encode.argtypes = [P, C.c_uint32, C.c_uint32, P, C.c_uint64, P, P]
        lib.refh_field_forward.argtypes = [P, C.c_uint32, C.c_uint32, P, P, P, C.c_uint64, P, P]
        lib.refh_field_backward.argtypes = [P, C.c_uint32, C.c_uint32, P, P, P, P, P, C.c_uint64]
        lib.refh_stage_grads.argtypes = [P, C.c_uint32, P, C.c_int]
        lib.refh_march_step.restype = C.c_double
        lib.refh_march_step.argtypes = [P]
        lib.refh_default_config.argtypes = [C.POINTER(RunConfig)]
        lib.refh_last_error.restype = C.c_char_p
        lib.refh_save_checkpoint.argtypes = [P, C.c_uint32, C.c_uint64, C.c_char_p]
        lib.refh_load_checkpoint.argtypes = [P, C.c_uint32, C.c_char_p, P]
        lib.refh_stage_bench.argtypes = [P, P, P, C.c_uint64, P, P, C.c_uint64, C.c_int, C.c_int, P]
        lib.refh_time_replicas.restype = C.c_double
        lib.refh_time_replicas.argtypes = [P, C.c_uint32, P, P, P, C.c_uint64, C.c_uint64,
                                           C.c_uint64]
        _ref = lib
    return _ref


class _RunBase:
    """Common numpy-facing API of the oracle run and the reference run."""

    def __init__(self, cfg, app_rows):
        self.cfg = cfg.copy()
        self.app = np.ascontiguousarray(np.asarray(app_rows, dtype=np.float64))
        self.n_images = self.app.shape[0]


class OracleRun(_RunBase):
    """or_run: single-threaded C restatement of DistributedRun (worker.cpp:630-834)."""

    def __init__(self, cfg, app_rows):
        super().__init__(cfg, app_rows)
        self.lib = oracle_lib()
        self.h = self.lib.or_run_create(C.byref(self.cfg), self.n_images, _ptr(self.app))
        if not self.h:
            raise RuntimeError(self.lib.or_last_error().decode())
        self.P = self.cfg.kx * self.cfg.ky
        self._nparams = [self._count(g) for g in range(self.P)]

    def _count(self, g):
        # parameter count from the reference layout formula (shared with the GPU layout)
        from paper_2405_04416_b200.layout import partition_param_count
        return partition_param_count(self.cfg, g)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.or_run_destroy(self.h)
            self.h = None

    def _arr(self, ptr, n):
        return np.ctypeslib.as_array(ptr, shape=(n,))

    def params(self, g):
        return self._arr(self.lib.or_run_params(self.h, g), self._nparams[g])

    def grads(self, g):
        return self._arr(self.lib.or_run_grads(self.h, g), self._nparams[g])

    def abs_grads(self, g):
        """sum over contributions of |contribution| for every gradient entry (last step)"""
        return self._arr(self.lib.or_run_abs_grads(self.h, g), self._nparams[g])

    def adam(self, g):
        m = self._arr(self.lib.or_run_adam_m(self.h, g), self._nparams[g])
        v = self._arr(self.lib.or_run_adam_v(self.h, g), self._nparams[g])
        return m, v, self.lib.or_run_adam_t(self.h, g)[0], self.lib.or_run_worker_step(self.h, g)[0]

    def set_params(self, g, p):
        self.params(g)[:] = p

    def set_adam(self, g, m, v, t, wstep):
        mm, vv, _, _ = self.adam(g)
        mm[:] = m
        vv[:] = v
        self.lib.or_run_adam_t(self.h, g)[0] = t
        self.lib.or_run_worker_step(self.h, g)[0] = wstep

    def set_occupancy(self, g, cascade, bits):
        bits = np.ascontiguousarray(bits, dtype=U8)
        self.lib.or_run_set_occupancy(self.h, g, cascade, _ptr(bits))

    def occupancy(self, g, cascade, ncells):
        return self._arr(self.lib.or_run_occ_bits(self.h, g, cascade), ncells).copy()

    def log_samples(self, g, capacity):
        """Record every training sample of partition g in the next train_step (test-only):
        sample_log() then returns (pos, features, field_out, upstream, d_features) in the GPU's
        dg_last_sample_data order."""
        self._slog = np.zeros((capacity, 96))
        self.lib.or_run_sample_log(self.h, g, _ptr(self._slog), capacity)

    def sample_log(self):
        n = int(self.lib.or_run_sample_log_count(self.h))
        L2 = 2 * self.cfg.grid_levels
        r = self._slog[:n]
        return r[:, 0:3], r[:, 3:3 + L2], r[:, 35:39], r[:, 39:43], r[:, 43:43 + L2]

    def mask_override(self, g, words):
        """Test-only: the ReLU decisions [n, 6] (h1 lo/hi, c1 lo/hi, c2 lo/hi 32-bit words) of
        partition g's training samples in the next train_step(s), in sample-log order (None: off).
        See gpu_mask_words for the GPU's mask layout."""
        keep = self.__dict__.setdefault("_movr", {})
        if words is None:
            keep.pop(g, None)
            self.lib.or_run_mask_override(self.h, g, None, 0)
            return
        keep[g] = np.ascontiguousarray(words, dtype=np.uint32)
        self.lib.or_run_mask_override(self.h, g, _ptr(keep[g]), len(words))

    def override_stats(self):
        """(units whose overridden decision went against the sign of z, their largest |z|) over
        the last train_step."""
        n, z = C.c_uint64(), C.c_double()
        self.lib.or_run_override_stats(self.h, C.byref(n), C.byref(z))
        return n.value, z.value

    def sample_log_masks(self):
        """ReLU signs (h1 lo/hi, c1 lo/hi, c2 lo/hi 32-bit words) and the smallest |pre-activation|
        of h1, c1, c2 per logged sample."""
        n = int(self.lib.or_run_sample_log_count(self.h))
        r = self._slog[:n]
        return r[:, 75:81].astype(np.uint32), r[:, 81:84]

    def train_step(self, o, d, gt, img, step):
        stats = np.zeros(8)
        gt64 = np.ascontiguousarray(gt, dtype=np.float64)
        img = np.ascontiguousarray(img, dtype=np.uint32)
        rc = self.lib.or_run_train_step(self.h, _ptr(o), _ptr(d), _ptr(gt64), _ptr(img), len(o),
                                        step, _ptr(stats))
        if rc != 0:
            raise RuntimeError(self.lib.or_last_error().decode())
        return dict(loss_rgb=stats[0], loss_transmittance=stats[1], loss_distortion=stats[2],
                    lr=stats[3], rays=int(stats[4]), dropped_rays=int(stats[5]))

    def eval_rays(self, o, d, app_vec):
        n = len(o)
        rgb = np.zeros((n, 3))
        T = np.zeros(n)
        depth = np.zeros(n)
        app_vec = np.ascontiguousarray(app_vec, dtype=np.float64)
        rc = self.lib.or_run_eval_rays(self.h, _ptr(o), _ptr(d), n, _ptr(app_vec), _ptr(rgb),
                                       _ptr(T), _ptr(depth))
        if rc != 0:
            raise RuntimeError(self.lib.or_last_error().decode())
        return rgb, T, depth

    def eval_rays_attribution(self, o, d, app_vec):
        n = len(o)
        rgb, T, depth, attr = np.zeros((n, 3)), np.zeros(n), np.zeros(n), np.zeros((n, 3))
        app_vec = np.ascontiguousarray(app_vec, dtype=np.float64)
        self.lib.or_run_eval_rays_ex.argtypes = [P, P, P, C.c_uint64, P, P, P, P, P]
        rc = self.lib.or_run_eval_rays_ex(self.h, _ptr(o), _ptr(d), n, _ptr(app_vec), _ptr(rgb),
                                          _ptr(T), _ptr(depth), _ptr(attr))
        if rc != 0:
            raise RuntimeError(self.lib.or_last_error().decode())
        return rgb, T, depth, attr


class RefRun(_RunBase):
    """The reference DistributedRun itself, through oracle/ref_harness.cpp."""

    def __init__(self, cfg, app_rows):
        super().__init__(cfg, app_rows)
        self.lib = ref_lib()
        self.h = self.lib.refh_create(C.byref(self.cfg), self.n_images, _ptr(self.app))
        if not self.h:
            raise RuntimeError(self.lib.refh_last_error().decode())
        self.P = self.cfg.kx * self.cfg.ky

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.refh_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.refh_last_error().decode())

    def nparams(self, g):
        return int(self.lib.refh_param_count(self.h, g))

    def stage_bench(self, o, d, pts, dirs, threads, bwd_threads):
        """Region 0's stage functions on a host thread pool (ref_harness.cpp refh_stage_bench)."""
        o, d = np.ascontiguousarray(o, np.float64), np.ascontiguousarray(d, np.float64)
        pts, dirs = np.ascontiguousarray(pts, np.float64), np.ascontiguousarray(dirs, np.float64)
        out = np.zeros(5)
        self._check(self.lib.refh_stage_bench(self.h, _ptr(o), _ptr(d), len(o), _ptr(pts), _ptr(dirs), len(pts),
                                              int(threads), int(bwd_threads), _ptr(out)))
        return {"segment_march_rays_per_s": out[0], "encode_samples_per_s": out[1],
                "field_fwd_samples_per_s": out[2], "field_bwd_samples_per_s": out[3],
                "adam_params_per_s": out[4]}

    def save_checkpoint(self, g, config_hash, path):
        self._check(self.lib.refh_save_checkpoint(self.h, g, config_hash, path.encode()))

    def load_checkpoint(self, g, path):
        h = C.c_uint64()
        self._check(self.lib.refh_load_checkpoint(self.h, g, path.encode(), C.byref(h)))
        return h.value

    def params(self, g):
        out = np.zeros(self.nparams(g))
        self.lib.refh_get_params(self.h, g, _ptr(out))
        return out

    def set_params(self, g, p):
        p = np.ascontiguousarray(p, dtype=np.float64)
        self.lib.refh_set_params(self.h, g, _ptr(p))

    def adam(self, g):
        n = self.nparams(g)
        m = np.zeros(n)
        v = np.zeros(n)
        t = C.c_uint64()
        ws = C.c_uint64()
        self.lib.refh_get_adam(self.h, g, _ptr(m), _ptr(v), C.byref(t), C.byref(ws))
        return m, v, t.value, ws.value

    def set_adam(self, g, m, v, t, wstep):
        m = np.ascontiguousarray(m, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        self._check(self.lib.refh_set_adam(self.h, g, _ptr(m), _ptr(v), t, wstep))

    def set_occupancy(self, g, cascade, bits):
        bits = np.ascontiguousarray(bits, dtype=U8)
        self.lib.refh_set_occupancy(self.h, g, cascade, _ptr(bits))

    def occupancy(self, g, cascade, ncells):
        bits = np.zeros(ncells, dtype=U8)
        self.lib.refh_get_occupancy(self.h, g, cascade, _ptr(bits), None)
        return bits

    def occupancy_density(self, g, cascade, ncells):
        den = np.zeros(ncells)
        bits = np.zeros(ncells, dtype=U8)
        self.lib.refh_get_occupancy(self.h, g, cascade, _ptr(bits), _ptr(den))
        return den

    def log_samples(self, g, capacity):
        """Record every training sample of partition g in the next train_step (test-only):
        sample_log() then returns (pos, features, field_out, upstream, d_features) in the GPU's
        dg_last_sample_data order."""
        self._slog = np.zeros((capacity, 96))
        self.lib.or_run_sample_log(self.h, g, _ptr(self._slog), capacity)

    def sample_log(self):
        n = int(self.lib.or_run_sample_log_count(self.h))
        L2 = 2 * self.cfg.grid_levels
        r = self._slog[:n]
        return r[:, 0:3], r[:, 3:3 + L2], r[:, 35:39], r[:, 39:43], r[:, 43:43 + L2]

    def mask_override(self, g, words):
        """Test-only: the ReLU decisions [n, 6] (h1 lo/hi, c1 lo/hi, c2 lo/hi 32-bit words) of
        partition g's training samples in the next train_step(s), in sample-log order (None: off).
        See gpu_mask_words for the GPU's mask layout."""
        keep = self.__dict__.setdefault("_movr", {})
        if words is None:
            keep.pop(g, None)
            self.lib.or_run_mask_override(self.h, g, None, 0)
            return
        keep[g] = np.ascontiguousarray(words, dtype=np.uint32)
        self.lib.or_run_mask_override(self.h, g, _ptr(keep[g]), len(words))

    def override_stats(self):
        """(units whose overridden decision went against the sign of z, their largest |z|) over
        the last train_step."""
        n, z = C.c_uint64(), C.c_double()
        self.lib.or_run_override_stats(self.h, C.byref(n), C.byref(z))
        return n.value, z.value

    def sample_log_masks(self):
        """ReLU signs (h1 lo/hi, c1 lo/hi, c2 lo/hi 32-bit words) and the smallest |pre-activation|
        of h1, c1, c2 per logged sample."""
        n = int(self.lib.or_run_sample_log_count(self.h))
        r = self._slog[:n]
        return r[:, 75:81].astype(np.uint32), r[:, 81:84]

    def train_step(self, o, d, gt, img, step):
        stats = np.zeros(8)
        gt64 = np.ascontiguousarray(gt, dtype=np.float64)
        img = np.ascontiguousarray(img, dtype=np.uint32)
        self._check(self.lib.refh_train_step(self.h, _ptr(o), _ptr(d), _ptr(gt64), _ptr(img),
                                             len(o), step, _ptr(stats)))
        return dict(loss_rgb=stats[0], loss_transmittance=stats[1], loss_distortion=stats[2],
                    lr=stats[3], rays=int(stats[4]), dropped_rays=int(stats[5]))

    def eval_rays(self, o, d, app_vec):
        n = len(o)
        rgb = np.zeros((n, 3))
        T = np.zeros(n)
        depth = np.zeros(n)
        app_vec = np.ascontiguousarray(app_vec, dtype=np.float64)
        self._check(self.lib.refh_eval_rays(self.h, _ptr(o), _ptr(d), n, _ptr(app_vec), _ptr(rgb),
                                            _ptr(T), _ptr(depth)))
        return rgb, T, depth

    def eval_image(self, camera, app_vec):
        """DistributedRun::evaluate_image for one camera dict -> (rgb, T, depth, attribution)."""
        from paper_2405_04416_b200.abi import cameras
        cam = cameras([camera])
        n = camera["width"] * camera["height"]
        rgb, T, depth, attr = np.zeros((n, 3)), np.zeros(n), np.zeros(n), np.zeros((n, 3))
        app_vec = np.ascontiguousarray(app_vec, dtype=np.float64)
        self.lib.refh_eval_image.argtypes = [P, P, P, P, P, P, P]
        self._check(self.lib.refh_eval_image(self.h, C.cast(cam, P), _ptr(app_vec), _ptr(rgb), _ptr(T),
                                             _ptr(depth), _ptr(attr)))
        return rgb, T, depth, attr

    # ---- stage functions ----
    def cascade_march(self, g, o, d, t0, t1, ray_id, jitter, batch_id, capacity=None):
        n = len(o)
        cap = capacity or int(n * 4096)
        counts = np.zeros(n, dtype=np.uint32)
        t = np.zeros(cap)
        delta = np.zeros(cap)
        casc = np.zeros(cap, dtype=U8)
        ray_id = np.ascontiguousarray(ray_id, dtype=np.uint64)
        self._check(self.lib.refh_cascade_march(self.h, g, _ptr(o), _ptr(d), _ptr(t0), _ptr(t1),
                                                _ptr(ray_id), n, int(jitter), batch_id,
                                                _ptr(counts), _ptr(t), _ptr(delta), _ptr(casc),
                                                cap))
        tot = int(counts.sum())
        return counts, t[:tot], delta[:tot], casc[:tot]

    def encode(self, g, cascade, pts):
        n = len(pts)
        L, F = self.cfg.grid_levels, self.cfg.grid_features
        out = np.zeros((n, L * F))
        rows = np.zeros((n, L, 8), dtype=np.uint32)
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        self._check(self.lib.refh_encode(self.h, g, cascade, _ptr(pts), n, _ptr(out), _ptr(rows)))
        return out, rows

    def field_forward(self, g, cascade, pts, dirs, app):
        n = len(pts)
        sigma = np.zeros(n)
        rgb = np.zeros((n, 3))
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        dirs = np.ascontiguousarray(dirs, dtype=np.float64)
        app = np.ascontiguousarray(app, dtype=np.float64)
        self._check(self.lib.refh_field_forward(self.h, g, cascade, _ptr(pts), _ptr(dirs),
                                                _ptr(app), n, _ptr(sigma), _ptr(rgb)))
        return sigma, rgb

    def field_backward(self, g, cascade, pts, dirs, app, dsig, drgb):
        n = len(pts)
        args = [np.ascontiguousarray(x, dtype=np.float64) for x in (pts, dirs, app, dsig, drgb)]
        self._check(self.lib.refh_field_backward(self.h, g, cascade, *[_ptr(a) for a in args], n))

    def stage_grads(self, g, zero=True):
        out = np.zeros(self.nparams(g))
        self.lib.refh_stage_grads(self.h, g, _ptr(out), int(zero))
        return out


def gpu_mask_words(masks):
    """The GPU's per-sample mask words [n, 7] (kernels_mlp_tc.cu k_mlp_fwd_tc: words 0-3 = h1 |
    c1 << 16 of 16-column part p, 4-5 = c2) -> the oracle's [n, 6] (h1, c1, c2 lo/hi)."""
    m = np.asarray(masks, dtype=np.uint64)
    lo16 = lambda w: m[:, w] & 0xffff
    hi16 = lambda w: m[:, w] >> 16
    out = np.stack([lo16(0) | (lo16(1) << 16), lo16(2) | (lo16(3) << 16),
                    hi16(0) | (hi16(1) << 16), hi16(2) | (hi16(3) << 16), m[:, 4], m[:, 5]], 1)
    return out.astype(np.uint32)


def ref_segment_rays(cfg, o, d):
    lib = ref_lib()
    n = len(o)
    nseg = np.zeros(n, dtype=U8)
    region = np.zeros((n, DG_MAX_SEGMENTS), dtype=np.uint16)
    te = np.zeros((n, DG_MAX_SEGMENTS))
    tx = np.zeros((n, DG_MAX_SEGMENTS))
    rc = lib.refh_segment_rays(C.byref(cfg), _ptr(o), _ptr(d), n, _ptr(nseg), _ptr(region),
                               _ptr(te), _ptr(tx))
    if rc != 0:
        raise RuntimeError(lib.refh_last_error().decode())
    return nseg, region, te, tx


def oracle_segment_rays(cfg, o, d):
    """or_segment_ray over a batch (partition.cpp:254-296 restated)."""
    lib = oracle_lib()
    model = ModelBuffer(cfg)
    n = len(o)
    nseg = np.zeros(n, dtype=U8)
    region = np.zeros((n, DG_MAX_SEGMENTS), dtype=np.uint32)
    te = np.zeros((n, DG_MAX_SEGMENTS))
    tx = np.zeros((n, DG_MAX_SEGMENTS))
    for i in range(n):
        k = lib.or_segment_ray(model.ptr, _ptr(o[i]), _ptr(d[i]),
                               region[i].ctypes.data_as(P), te[i].ctypes.data_as(P),
                               tx[i].ctypes.data_as(P))
        nseg[i] = k
    return nseg, region.astype(np.uint16), te, tx


class ModelBuffer:
    """An or_model initialised for cfg (opaque, sized generously)."""

    SIZE = 1 << 20

    def __init__(self, cfg):
        lib = oracle_lib()
        self.buf = C.create_string_buffer(self.SIZE)
        self.cfg = cfg.copy()
        lib.or_model_init.argtypes = [P, C.POINTER(RunConfig)]
        rc = lib.or_model_init(C.cast(self.buf, P), C.byref(self.cfg))
        if rc != 0:
            raise RuntimeError(lib.or_last_error().decode())
        self.ptr = C.cast(self.buf, P)


class OracleModel:
    """or_model for cfg + the per-stage restatements on flat partition arrays."""

    def __init__(self, cfg):
        lib = oracle_lib()
        lib.or_model_size.restype = C.c_uint64
        lib.or_model_init.argtypes = [P, C.POINTER(RunConfig)]
        self.cfg = cfg.copy()
        self.buf = C.create_string_buffer(int(lib.or_model_size()))
        self.ptr = C.cast(self.buf, P)
        if lib.or_model_init(self.ptr, C.byref(self.cfg)) != 0:
            raise RuntimeError(lib.or_last_error().decode())
        self.lib = lib
        lib.or_stage_cascade_march.argtypes = [P, C.c_uint32, P, P, P, P, P, P, P, C.c_uint64,
                                               C.c_int, C.c_uint64, P, P, P, P, C.c_uint64]
        lib.or_stage_encode.argtypes = [P, C.c_uint32, C.c_uint32, P, P, C.c_uint64, P, P]
        lib.or_stage_field_forward.argtypes = [P, C.c_uint32, C.c_uint32, P, P, P, P, C.c_uint64,
                                               P, P]
        lib.or_stage_field_backward.argtypes = [P, C.c_uint32, C.c_uint32, P, P, P, P, P, P, P,
                                                C.c_uint64]
        lib.or_segment_ray.argtypes = [P, P, P, P, P, P]

    def segment_rays(self, o, d):
        n = len(o)
        nseg = np.zeros(n, dtype=U8)
        region = np.zeros((n, DG_MAX_SEGMENTS), dtype=np.uint32)
        te = np.zeros((n, DG_MAX_SEGMENTS))
        tx = np.zeros((n, DG_MAX_SEGMENTS))
        o = np.ascontiguousarray(o, dtype=np.float64)
        d = np.ascontiguousarray(d, dtype=np.float64)
        for i in range(n):
            nseg[i] = self.lib.or_segment_ray(self.ptr, _ptr(o[i]), _ptr(d[i]), _ptr(region[i]),
                                              _ptr(te[i]), _ptr(tx[i]))
        return nseg, region.astype(np.uint16), te, tx

    def cascade_march(self, g, occ_fine, occ_coarse, o, d, t0, t1, ray_id, jitter, batch_id):
        n = len(o)
        cap = max(16, int(n) * 8192)
        counts = np.zeros(n, dtype=np.uint32)
        t = np.zeros(cap)
        delta = np.zeros(cap)
        casc = np.zeros(cap, dtype=U8)
        args = [np.ascontiguousarray(x, dtype=np.float64) for x in (o, d, t0, t1)]
        rid = np.ascontiguousarray(ray_id, dtype=np.uint64)
        of = np.ascontiguousarray(occ_fine, dtype=U8)
        oc = np.ascontiguousarray(occ_coarse, dtype=U8)
        rc = self.lib.or_stage_cascade_march(self.ptr, g, _ptr(of), _ptr(oc), *[_ptr(a) for a in args],
                                             _ptr(rid), n, int(jitter), batch_id, _ptr(counts),
                                             _ptr(t), _ptr(delta), _ptr(casc), cap)
        if rc != 0:
            raise RuntimeError(self.lib.or_last_error().decode())
        tot = int(counts.sum())
        return counts, t[:tot], delta[:tot], casc[:tot]

    def encode(self, g, cascade, params, pts):
        n = len(pts)
        L, F = self.cfg.grid_levels, self.cfg.grid_features
        out = np.zeros((n, L * F))
        rows = np.zeros((n, L, 8), dtype=np.uint32)
        params = np.ascontiguousarray(params, dtype=np.float64)
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        self.lib.or_stage_encode(self.ptr, g, cascade, _ptr(params), _ptr(pts), n, _ptr(out),
                                 _ptr(rows))
        return out, rows

    def encode_rows(self, g, cascade, pts):
        """Hash-table rows only (no tables needed, any table size)."""
        n = len(pts)
        out = np.zeros((n, self.cfg.grid_levels * self.cfg.grid_features))
        rows = np.zeros((n, self.cfg.grid_levels, 8), dtype=np.uint32)
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        self.lib.or_stage_encode(self.ptr, g, cascade, None, _ptr(pts), n, _ptr(out), _ptr(rows))
        return rows

    def field_forward(self, g, cascade, params, pts, dirs, app):
        n = len(pts)
        sigma = np.zeros(n)
        rgb = np.zeros((n, 3))
        a = [np.ascontiguousarray(x, dtype=np.float64) for x in (params, pts, dirs, app)]
        self.lib.or_stage_field_forward(self.ptr, g, cascade, *[_ptr(x) for x in a], n,
                                        _ptr(sigma), _ptr(rgb))
        return sigma, rgb

    def field_backward(self, g, cascade, params, pts, dirs, app, dsig, drgb):
        n = len(pts)
        params = np.ascontiguousarray(params, dtype=np.float64)
        grads = np.zeros_like(params)
        a = [np.ascontiguousarray(x, dtype=np.float64) for x in (pts, dirs, app, dsig, drgb)]
        self.lib.or_stage_field_backward(self.ptr, g, cascade, _ptr(params), _ptr(grads),
                                         *[_ptr(x) for x in a], n)
        return grads


# ---- ray cache: C restatement and the reference's own RayCache ----
class _CacheBase:
    def __init__(self, poses, images, capacity, seed):
        from paper_2405_04416_b200.abi import cameras
        self._cams = cameras(poses)
        self._imgs = [np.ascontiguousarray(im, dtype=np.uint8) for im in images]
        self._ptrs = (C.c_void_p * len(self._imgs))(*[im.ctypes.data for im in self._imgs])

    @staticmethod
    def _bufs(n):
        return (np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n, np.uint32),
                np.zeros(n, np.uint64))


class OracleRayCache(_CacheBase):
    def __init__(self, poses, images, capacity, seed):
        super().__init__(poses, images, capacity, seed)
        L = oracle_lib()
        L.or_ray_cache_create.restype = P
        L.or_ray_cache_create.argtypes = [P, P, C.c_uint32, C.c_uint64, C.c_uint64]
        L.or_ray_cache_destroy.argtypes = [P]
        L.or_ray_cache_size.restype = C.c_uint64
        L.or_ray_cache_size.argtypes = [P]
        L.or_ray_cache_refresh.argtypes = [P, C.c_uint64]
        L.or_ray_cache_draw.argtypes = [P, C.c_uint64, P, P, P, P, P]
        L.or_ray_cache_snapshot.argtypes = [P, P, P, P, P, P]
        self.L = L
        self.h = L.or_ray_cache_create(C.cast(self._cams, P), C.cast(self._ptrs, P), len(self._imgs),
                                       capacity, seed)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.or_ray_cache_destroy(self.h)
            self.h = None

    def size(self):
        return self.L.or_ray_cache_size(self.h)

    def refresh(self, count):
        assert self.L.or_ray_cache_refresh(self.h, count) == 0

    def draw(self, n):
        out = self._bufs(n)
        assert self.L.or_ray_cache_draw(self.h, n, *[_ptr(a) for a in out]) == 0
        return out

    def snapshot(self):
        out = self._bufs(self.size())
        self.L.or_ray_cache_snapshot(self.h, *[_ptr(a) for a in out])
        return out


class RefRayCache(_CacheBase):
    def __init__(self, poses, images, capacity, seed):
        super().__init__(poses, images, capacity, seed)
        L = ref_lib()
        L.refh_ray_cache_create.restype = P
        L.refh_ray_cache_create.argtypes = [P, P, C.c_uint32, C.c_uint64, C.c_uint64]
        L.refh_ray_cache_destroy.argtypes = [P]
        L.refh_ray_cache_refresh.argtypes = [P, C.c_uint64]
        L.refh_ray_cache_snapshot.restype = C.c_uint64
        L.refh_ray_cache_snapshot.argtypes = [P, P, P, P, P, P]
        L.refh_ray_cache_draw.argtypes = [P, C.c_uint64, P, P, P, P, P]
        self.L = L
        self.h = L.refh_ray_cache_create(C.cast(self._cams, P), C.cast(self._ptrs, P), len(self._imgs),
                                         capacity, seed)
        assert self.h, L.refh_last_error()

    def __del__(self):
        if getattr(self, "h", None):
            self.L.refh_ray_cache_destroy(self.h)
            self.h = None

    def size(self):
        return int(self.L.refh_ray_cache_snapshot(self.h, None, None, None, None, None))

    def refresh(self, count):
        assert self.L.refh_ray_cache_refresh(self.h, count) == 0, self.L.refh_last_error()

    def draw(self, n):
        out = self._bufs(n)
        assert self.L.refh_ray_cache_draw(self.h, n, *[_ptr(a) for a in out]) == 0, self.L.refh_last_error()
        return out

    def snapshot(self):
        out = self._bufs(self.size())
        self.L.refh_ray_cache_snapshot(self.h, *[_ptr(a) for a in out])
        return out
