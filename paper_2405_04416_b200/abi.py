"""ctypes mirrors of the C structs in include/distgrid_b200.h (no library loading here).

Kept separate so that the test-only oracle bindings can share the config layout with the
product binding (paper_2405_04416_b200/dg.py) without importing the CUDA library.
"""
import ctypes as C

import numpy as np

DG_MAX_SEGMENTS = 16
DG_MAX_PARTITIONS = 64
DG_MAX_LEVELS = 16
DG_MEM_HOST = 0
DG_MEM_DEVICE = 1

STATUS_NAMES = {0: "DG_OK", 1: "DG_EINVAL", 2: "DG_ERANGE", 3: "DG_EPROTO",
                4: "DG_ETIMEOUT", 5: "DG_ECUDA", 6: "DG_ENCCL", 7: "DG_ENOMEM"}


class RunConfig(C.Structure):
    """dg_run_config: RunConfig (config.hpp:13-78) + split_regions boxes."""
    _fields_ = [
        ("inner_lo", C.c_double * 3), ("inner_hi", C.c_double * 3),
        ("outer_lo", C.c_double * 3), ("outer_hi", C.c_double * 3),
        ("ground_altitude", C.c_double),
        ("kx", C.c_uint32), ("ky", C.c_uint32),
        ("grid_levels", C.c_uint32), ("grid_features", C.c_uint32),
        ("base_resolution", C.c_uint32), ("max_resolution", C.c_uint32),
        ("fine_table_log2", C.c_uint32), ("coarse_table_log2", C.c_uint32),
        ("appearance_dim", C.c_uint32),
        ("march_step_divisor", C.c_double),
        ("occ_resolution", C.c_uint32), ("occ_decay", C.c_double),
        ("occ_warmup_steps", C.c_uint64), ("occ_update_interval", C.c_uint64),
        ("occ_threshold_early", C.c_double), ("occ_threshold_late", C.c_double),
        ("occ_threshold_switch_step", C.c_uint64), ("occ_threshold_scale", C.c_double),
        ("seed", C.c_uint64), ("total_steps", C.c_uint64),
        ("lr_start", C.c_double), ("lr_end", C.c_double),
        ("lambda_transmittance", C.c_double), ("lambda_distortion", C.c_double),
        ("transmittance_clamp", C.c_double),
        ("adam_beta1", C.c_double), ("adam_beta2", C.c_double), ("adam_eps", C.c_double),
        ("wire_f32", C.c_uint32), ("distortion_cross_correction", C.c_uint32),
        ("occupancy_updates", C.c_uint32), ("eval_early_termination", C.c_uint32),
        ("eval_termination_threshold", C.c_double),
    ]

    def copy(self):
        c = RunConfig()
        C.memmove(C.byref(c), C.byref(self), C.sizeof(RunConfig))
        return c

    def as_dict(self):
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = list(v) if hasattr(v, "__len__") else v
        return out


class RayBatch(C.Structure):
    _fields_ = [("origin", C.c_void_p), ("dir", C.c_void_p), ("color_gt", C.c_void_p),
                ("image_id", C.c_void_p), ("n", C.c_uint64), ("first_ray_id", C.c_uint64),
                ("mem", C.c_int32), ("reserved", C.c_int32)]


class StepStats(C.Structure):
    _fields_ = [("step", C.c_uint64), ("loss_rgb", C.c_double),
                ("loss_transmittance", C.c_double), ("loss_distortion", C.c_double),
                ("lr", C.c_double), ("rays", C.c_uint64), ("dropped_rays", C.c_uint64),
                ("bytes_sent", C.c_uint64), ("samples", C.c_uint64), ("items", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("partial_bytes_sent", C.c_uint64), ("partial_records_sent", C.c_uint64)]


class Merged(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("transmittance", C.c_void_p), ("depth", C.c_void_p),
                ("attribution", C.c_void_p), ("mem", C.c_int32), ("reserved", C.c_int32)]


class ArrayDesc(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("size", C.c_uint64), ("cascade", C.c_uint32),
                ("kind", C.c_uint32), ("index", C.c_uint32), ("reserved", C.c_uint32)]


class ItemView(C.Structure):
    _fields_ = [("n_items", C.c_uint64), ("n_fine", C.c_uint64), ("n_coarse", C.c_uint64)]


class Camera(C.Structure):
    """dg_camera: CameraPose (partition.hpp:15-28) + split flag."""
    _fields_ = [("image_id", C.c_uint32), ("width", C.c_uint32), ("height", C.c_uint32),
                ("is_train", C.c_uint32), ("rotation", C.c_double * 9), ("translation", C.c_double * 3),
                ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double)]


def cameras(poses):
    """Array of Camera from dicts {image_id, width, height, is_train, rotation (3x3), translation, fx, fy, cx, cy}."""
    arr = (Camera * len(poses))()
    for i, p in enumerate(poses):
        c = arr[i]
        c.image_id, c.width, c.height, c.is_train = p["image_id"], p["width"], p["height"], int(p["is_train"])
        for j, v in enumerate(list(np.asarray(p["rotation"], dtype=np.float64).reshape(9))):
            c.rotation[j] = float(v)
        for j in range(3):
            c.translation[j] = float(p["translation"][j])
        c.fx, c.fy, c.cx, c.cy = (float(p[k]) for k in ("fx", "fy", "cx", "cy"))
    return arr


class StageTimes(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("segment", "march", "encode_fwd", "mlp_fwd", "composite",
                                         "exchange", "merge_bwd", "mlp_bwd", "encode_bwd",
                                         "adam", "total", "dispatch_exchange", "dispatch_mb",
                                         "partial_mb")] + [("reserved", C.c_float * 2)]

    def as_dict(self):
        return {n: float(getattr(self, n)) for n, _ in self._fields_ if n != "reserved"}


def default_config():
    """RunConfig defaults (config.hpp:13-78; train.hpp:14-18, 50-54), inner = outer = [0,1]^3."""
    c = RunConfig()
    for a in range(3):
        c.inner_lo[a] = c.outer_lo[a] = 0.0
        c.inner_hi[a] = c.outer_hi[a] = 1.0
    c.ground_altitude = 0.0
    c.kx = c.ky = 1
    c.grid_levels = 8
    c.grid_features = 2
    c.base_resolution = 16
    c.max_resolution = 512
    c.fine_table_log2 = 15
    c.coarse_table_log2 = 12
    c.appearance_dim = 16
    c.march_step_divisor = 1024.0
    c.occ_resolution = 128
    c.occ_decay = 0.99
    c.occ_warmup_steps = 4096
    c.occ_update_interval = 16
    c.occ_threshold_early = 0.6
    c.occ_threshold_late = 60.0
    c.occ_threshold_switch_step = 10000
    c.occ_threshold_scale = 1.0
    c.seed = 1
    c.total_steps = 20000
    c.lr_start = 0.05
    c.lr_end = 0.005
    c.lambda_transmittance = 1e-3
    c.lambda_distortion = 1e-3
    c.transmittance_clamp = 1e-6
    c.adam_beta1 = 0.9
    c.adam_beta2 = 0.99
    c.adam_eps = 1e-15
    c.wire_f32 = 0
    c.distortion_cross_correction = 0
    c.occupancy_updates = 1
    c.eval_early_termination = 0
    c.eval_termination_threshold = 1e-4
    return c
