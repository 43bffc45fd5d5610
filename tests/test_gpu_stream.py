"""dg_set_stream: every call of a context runs on the caller's CUDA stream (the
stage calls take the caller's cudaStream_t).  A training step on a torch-created stream gives
the losses of the same step on the context's own stream, and the stream really is the one
used (an event recorded on it after the step completes only once the step's work is done)."""
import numpy as np
import pytest
import torch

from paper_2405_04416_b200 import dg, workloads

from .helpers import app_rows, inject, small_cfg

pytestmark = pytest.mark.gpu


def _run(stream):
    cfg = small_cfg(2, 1, table_log2=12, levels=6, nmax=128, divisor=48)
    ctx = dg.Context(cfg, device=0)
    inject(cfg, ctx, [], occupancy_fraction=0.7)
    ctx.set_appearance(app_rows(1).astype(np.float32))
    own = ctx.stream()
    if stream is not None:
        ctx.set_stream(stream.cuda_stream)
        assert ctx.stream() == stream.cuda_stream
    o, d, gt, img = workloads.make_rays(cfg, 2000, "independent", seed=9)
    st = ctx.train_step(o, d, gt, img, step=0)
    if stream is not None:
        ev = torch.cuda.Event()
        ev.record(stream)
        ev.synchronize()
        ctx.set_stream(None)
        assert ctx.stream() == own
    return st


def test_train_step_on_caller_stream():
    a = _run(None)
    b = _run(torch.cuda.Stream())
    for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
        assert abs(a[k] - b[k]) <= 1e-6 * abs(a[k]) + 1e-12, (k, a[k], b[k])
    assert a["samples"] == b["samples"]
