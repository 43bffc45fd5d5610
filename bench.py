#!/usr/bin/env python
"""bench.py — training rays/s (and render rays/s, encode GB/s) of the B200 DistGrid path.

Contract (see the task statement): `python bench.py --gpus N --steps K --warmup W` runs the
training step on N GPUs of one node (torchrun for N > 1, one rank per GPU, one partition per
GPU), times exactly K steps after W warm-up steps with CUDA events on the step stream,
bracketed by barrier + synchronize, max over ranks, and rank 0 prints ONE JSON line.

Workload (SURVEY §8d weak-scaling point of C4): G = N partitions in a kx x ky tiling of unit
tiles (1x1, 2x1, 2x2, 4x2), hash grid L=16 F=2 T=2^24 per partition, N0=16, Nmax=2048,
131,072 rays per GPU from the balanced reflected-drift generator, march step 4/416
(~128 samples/ray), inner == outer box, occupancy all occupied, random-init parameters.
A step = DistributedRun::training_step over the whole batch: segmentation, dispatch,
march, encode, MLP, composite, partial exchange, merge + losses + backward, dense Adam.

`--impl reference` times the reference's own CPU implementation (oracle/_ref, the
unmodified reference library) on this host, rank 0 only.
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training rays/sec and render rays/sec at 1/2/4/8 B200; encode GB/s vs HBM/L2 peak"
ENCODE_BYTES_PER_SAMPLE = 16 * 8 * 2 * 4      # L x 8 corners x F x fp32
MLP_FLOP_TRAIN = 62208                          # fwd + bwd per sample


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops_sustained"]), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback"


def profile_traffic():
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the hot kernels,
    from the committed ncu --set full capture summarised in profiles/traffic.json."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return {k: v["dram_bytes_per_launch"] for k, v in json.load(f)["kernels"].items()}
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 2 + k and s[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ reference arm
def host_cpu():
    import os
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return n, model


def cpu_stage_baseline(run, o, d):
    """the reference's stage functions (segment_ray + cascade_march, encode,
    query_density + query_color, field_backward incl. encode_backward, AdamState::step) on a
    std::thread pool over every host core.  The backward gives each thread its own FieldGrads
    sink (a full table-shaped copy), so its thread count is capped by host memory."""
    nproc, model = host_cpu()
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    sink = run.nparams(0) * 8
    bwd_threads = int(max(1, min(nproc, (0.4 * avail) // max(sink, 1))))
    rng = np.random.default_rng(11)
    n_pts = 65536
    pts = rng.uniform(0.0, 1.0, (n_pts, 3))
    dirs = rng.normal(size=(n_pts, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    t0 = time.perf_counter()
    run.stage_bench(o[:1024], d[:1024], pts[:4096], dirs[:4096], nproc, bwd_threads)  # warm-up (page-in)
    res = run.stage_bench(o, d, pts, dirs, nproc, bwd_threads)
    res.update({"threads": nproc, "bwd_threads": bwd_threads, "cpu": model,
                "sample": f"{len(o)} rays (segment+march), {n_pts} uniform points (encode / field), "
                          f"one Adam step over the fine field; wall {time.perf_counter() - t0:.1f}s"})
    return res


def cpu_reference(cfg, o, d, gt, rays, steps, warmup, stages=False):
    """The unmodified reference DistributedRun (oracle/_ref) on this host: each step is a
    bounded sample of `rays` rays of the same workload (its K=1 worker thread + driver)."""
    from oracle.bindings import RefRun, ref_available
    from paper_2405_04416_b200 import workloads
    if not ref_available():
        return None, "oracle/_ref not built"
    app = workloads.appearance_rows(cfg.appearance_dim, 1)
    t0 = time.perf_counter()
    run = RefRun(cfg, app)
    init_s = time.perf_counter() - t0
    img = np.zeros(rays, dtype=np.uint32)
    times = []
    for s in range(warmup + steps):
        lo = (s * rays) % max(1, len(o) - rays)
        a = time.perf_counter()
        run.train_step(o[lo:lo + rays], d[lo:lo + rays], gt[lo:lo + rays].astype(np.float64), img, s)
        if s >= warmup:
            times.append(time.perf_counter() - a)
    stage = None
    if stages:
        try:
            stage = cpu_stage_baseline(run, o, d)
        except Exception as e:  # the headline baseline stands without it
            stage = {"unavailable": str(e)[:200]}
    del run
    sec = float(np.sum(times))
    return {"value": rays * len(times) / sec, "unit": "rays/s", "cores": 1, "kind": "reference",
            "sample": f"{len(times)} x DistributedRun::training_step on {rays} rays of the bench "
                      f"workload (K=1 worker thread; reference init {init_s:.1f}s excluded)",
            "ms_per_step": 1000 * sec / len(times), "stages": stage}, None


REF_REPLICA_BYTES = 11.5e9  # one reference DistributedRun at T = 2^24 (tools/diag/ref_rss.py: 10.7 GB)


def cpu_reference_replicas(cfg, rays, steps, warmup, generator):
    """All host threads the reference can use: it parallelises only across partitions (one
    worker thread each), so at the 1-GPU point (K = 1) the host runs independent replicas of
    the reference DistributedRun, one per thread, each training on its own ray slice in lock
    step (ref_harness.cpp refh_time_replicas).  The replica count is capped by host memory."""
    import ctypes as C
    from concurrent.futures import ThreadPoolExecutor

    from oracle.bindings import RefRun, ref_available, ref_lib
    from paper_2405_04416_b200 import workloads
    if not ref_available():
        return None, "oracle/_ref not built"
    nproc, model = host_cpu()
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32e9
    per = REF_REPLICA_BYTES * (1 << max(0, cfg.fine_table_log2 - 24)) if cfg.fine_table_log2 >= 24 else 2e9
    n_rep = int(max(1, min(nproc, (0.45 * avail) // per)))
    o, d, gt, _ = workloads.make_rays(cfg, n_rep * rays, generator, seed=1)
    app = workloads.appearance_rows(cfg.appearance_dim, 1)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(n_rep) as ex:  # refh_create runs without the GIL
        runs = list(ex.map(lambda _: RefRun(cfg, app), range(n_rep)))
    init_s = time.perf_counter() - t0
    lib = ref_lib()
    handles = (C.c_void_p * n_rep)(*[r.h for r in runs])
    o, d, gt = (np.ascontiguousarray(x, np.float64) for x in (o, d, gt))
    args = (handles, n_rep, o.ctypes.data_as(C.c_void_p), d.ctypes.data_as(C.c_void_p),
            gt.ctypes.data_as(C.c_void_p), rays)
    if warmup and lib.refh_time_replicas(*args, warmup, 0) < 0:
        return None, lib.refh_last_error().decode()
    sec = lib.refh_time_replicas(*args, steps, warmup)
    if sec < 0:
        return None, lib.refh_last_error().decode()
    del runs
    value = n_rep * rays * steps / sec
    return {"value": value, "unit": "rays/s", "cores": n_rep, "kind": "reference",
            "sample": f"{n_rep} replicas of the reference DistributedRun (K=1 worker thread each; "
                      f"the reference parallelises only across partitions), {rays} rays/step each, "
                      f"{steps} lock-step steps; {nproc}-thread host ({model}); init {init_s:.1f}s excluded",
            "ms_per_step": 1000 * sec / steps}, None


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from paper_2405_04416_b200 import workloads
    wl = workloads.weak(1, rays_per_gpu=args.rays_per_gpu, table_log2=args.table_log2)
    res, why = cpu_reference_replicas(wl.cfg, args.ref_rays, args.steps, min(args.warmup, 1), wl.generator)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": why}))
        return 0
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": "rays/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.name + " (CPU sample)", "rays_per_step_per_replica": args.ref_rays,
                       "table_log2": args.table_log2, "partitions": 1},
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": res["value"], "unit": "rays/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)  # = occ_update_interval: one update amortised
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rays-per-gpu", type=int, default=131072)
    ap.add_argument("--table-log2", type=int, default=24)
    ap.add_argument("--render-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="weak", choices=["weak", "C1", "C2", "C3", "C4", "C5"],
                    help="weak: the C4 weak-scaling point (default); C1..C5: a BASELINE config whole")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "peer"],
                    help="exchange backend for N > 1: NCCL all-to-all-v, or peer-memory pack kernels")
    ap.add_argument("--no-cpu-stages", action="store_true", help="skip the all-core stage baseline")
    ap.add_argument("--ref-rays", type=int, default=1024, help="rays per step per replica of the --impl reference arm")
    ap.add_argument("--cpu-rays", type=int, default=2048, help="rays of the cpu_baseline sample (~10 s)")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    from paper_2405_04416_b200 import abi, dg, workloads

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    if args.workload == "weak":
        wl = workloads.weak(world, rays_per_gpu=args.rays_per_gpu, table_log2=args.table_log2)
    else:  # a BASELINE config as a whole on `world` GPUs (partition p on rank p % world)
        wl = workloads.by_name(args.workload)
        args.no_cpu = True
    cfg = wl.cfg
    B = wl.n_rays
    shard = B // world
    lo, hi = rank * shard, (rank + 1) * shard
    NB = 1 if args.profile else 3  # distinct batches cycled over the steps
    batches_host = []
    for k in range(NB):
        o, d, gt, img = workloads.make_rays(cfg, B, wl.generator, seed=1 + k)
        batches_host.append((o[lo:hi], d[lo:hi], gt[lo:hi], img[lo:hi]))

    ctx = dg.Context(cfg, device=local, rank=rank, world=world)
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.tensor(list(dg.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        if args.comm == "peer":  # pack kernels write the owners' buffers over CUDA IPC
            gloo = dist.new_group(backend="gloo")

            def allgather(blob):
                out = [None] * world
                dist.all_gather_object(out, blob, group=gloo)
                return out

            ctx.comm_init_peer(allgather)
        else:
            ctx.comm_init_nccl(bytes(uid.cpu().tolist()))
    for g in ctx.local:
        ctx.init_fast(g, seed=1)
    ctx.set_appearance(workloads.appearance_rows(cfg.appearance_dim, 1))

    # device-resident inputs (value) ---------------------------------------------
    dev = []
    for (o, d, gt, img) in batches_host:
        t = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (o, d, gt, img.astype(np.int32))]
        b = abi.RayBatch()
        b.origin, b.dir, b.color_gt, b.image_id = (t[0].data_ptr(), t[1].data_ptr(),
                                                   t[2].data_ptr(), t[3].data_ptr())
        b.n, b.first_ray_id, b.mem = len(o), lo, abi.DG_MEM_DEVICE
        dev.append((b, t))
    sptr = C.c_void_p()
    dg.lib().dg_get_stream(ctx.h, C.byref(sptr))
    stream = torch.cuda.ExternalStream(sptr.value)
    stats = abi.StepStats()

    def step(i, batches):
        rc = ctx.train_step_raw(batches[i % len(batches)][0], i, stats)
        if rc != 0:
            raise dg.DGError(rc, dg.lib().dg_last_error().decode())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, n, first):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(n):
            fn(first + i)
        e1.record(stream)
        e1.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    for i in range(args.warmup):
        step(i, dev)
    launches0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        ms = timed(lambda i: step(i, dev), args.steps, args.warmup)
    launches = ctx.kernel_launches() - launches0
    ms_per_step = ms / args.steps
    value = B / (ms_per_step / 1000.0)
    samples_rank = int(stats.samples)
    items_rank = int(stats.items)
    bytes_sent = int(stats.bytes_sent)

    # per-stage device times of one more step (events on the step stream)
    ctx.enable_stage_timing(True)
    step(args.warmup + args.steps, dev)
    st = ctx.stage_times()
    ctx.enable_stage_timing(False)

    line = None
    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_per_step, "stages_ms": st}))
        if world > 1:
            dist.destroy_process_group()
        return 0

    # render throughput (evaluate_rays through the same kernels) ------------------
    m = abi.Merged()
    out = [torch.empty(x, device="cuda") for x in ((shard, 3), (shard,), (shard,))]
    m.rgb, m.transmittance, m.depth, m.mem = (out[0].data_ptr(), out[1].data_ptr(),
                                               out[2].data_ptr(), abi.DG_MEM_DEVICE)
    app = np.ascontiguousarray(workloads.appearance_rows(cfg.appearance_dim, 1)[0], dtype=np.float32)

    def render(i):
        rc = ctx.render_raw(dev[i % len(dev)][0], app, m)
        if rc != 0:
            raise dg.DGError(rc, dg.lib().dg_last_error().decode())

    render(0)
    rms = timed(render, args.render_steps, 0) / args.render_steps
    render_value = B / (rms / 1000.0)

    # end-to-end through the C ABI with pinned host buffers -------------------------
    e2e = None
    if not args.no_e2e:
        pinned = []
        for (o, d, gt, img) in batches_host:
            t = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (o, d, gt, img.astype(np.int32))]
            b = abi.RayBatch()
            b.origin, b.dir, b.color_gt, b.image_id = (t[0].data_ptr(), t[1].data_ptr(),
                                                       t[2].data_ptr(), t[3].data_ptr())
            b.n, b.first_ray_id, b.mem = len(o), lo, abi.DG_MEM_HOST
            pinned.append((b, t))
        step(0, pinned)
        ems = timed(lambda i: step(i, pinned), args.steps, args.warmup + args.steps + 1)
        e2e = {"value": B / (ems / args.steps / 1000.0), "unit": "rays/s",
               "h2d_bytes_per_step": int(stats.h2d_bytes), "d2h_bytes_per_step": int(stats.d2h_bytes),
               "ms_per_step": ems / args.steps}

    # roofline of the dominant kernel + the encode kernels ----------------------------
    hbm, tensor_peak, peak_kind = peaks()
    enc_bytes = samples_rank * ENCODE_BYTES_PER_SAMPLE
    stage_ms = {k: v for k, v in st.items() if k != "total"}
    dominant = max(stage_ms, key=stage_ms.get)
    enc_fwd_gbs = enc_bytes / (st["encode_fwd"] / 1e3) / 1e9 if st["encode_fwd"] > 0 else 0.0
    enc_bwd_gbs = 2 * enc_bytes / (st["encode_bwd"] / 1e3) / 1e9 if st["encode_bwd"] > 0 else 0.0
    mlp_tflops = samples_rank * MLP_FLOP_TRAIN / ((st["mlp_fwd"] + st["mlp_bwd"]) / 1e3) / 1e12
    traffic = profile_traffic()
    if dominant in ("mlp_fwd", "mlp_bwd"):
        roof = {"kernel": "k_mlp_fwd_tc+k_mlp_bwd_tc", "bound": "tensor", "achieved": mlp_tflops,
                "peak": tensor_peak, "unit": "TFLOP/s", "frac": mlp_tflops / tensor_peak,
                "traffic": traffic.get("k_mlp_bwd_tc"),
                "note": f"{MLP_FLOP_TRAIN} algorithmic FLOP/sample x {samples_rank} samples; the "
                        f"tcgen05 split-bf16 kernels execute 3 bf16 MMAs per product; peak = "
                        f"{peak_kind} sustained dense bf16"}
    else:
        ach = {"encode_fwd": enc_fwd_gbs, "encode_bwd": enc_bwd_gbs}.get(dominant, enc_fwd_gbs)
        kname = {"encode_fwd": "k_encode_fwd", "encode_bwd": "k_encode_bwd"}.get(dominant, dominant)
        roof = {"kernel": kname, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": traffic.get(kname),
                "note": "achieved = algorithmic bytes (SURVEY 8d) / the kernel's live CUDA-event time; "
                        "traffic = DRAM read+write bytes per launch from the committed ncu --set full "
                        "capture (profiles/traffic.json)"}
    roof["stage_ms"] = st
    # every hot kernel against its own roof (the dominant stage above can flip between the
    # MLP backward and the encoding backward from run to run)
    n_par = sum(ctx.param_count(g) for g in ctx.local)
    adam_gbs = 32.0 * n_par / (st["adam"] / 1e3) / 1e9 if st["adam"] > 0 else 0.0
    roofline_kernels = {
        "k_encode_fwd": {"bound": "hbm", "achieved": enc_fwd_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": enc_fwd_gbs / hbm, "traffic": traffic.get("k_encode_fwd"),
                         "algorithmic": f"{ENCODE_BYTES_PER_SAMPLE} B/sample"},
        "k_encode_bwd": {"bound": "hbm (L2 atomics)", "achieved": enc_bwd_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": enc_bwd_gbs / hbm, "traffic": traffic.get("k_encode_bwd"),
                         "algorithmic": f"{2 * ENCODE_BYTES_PER_SAMPLE} B/sample (RMW)"},
        "k_mlp_fwd_tc+k_mlp_bwd_tc": {"bound": "tensor", "achieved": mlp_tflops, "peak": tensor_peak,
                                      "unit": "TFLOP/s", "frac": mlp_tflops / tensor_peak,
                                      "traffic": traffic.get("k_mlp_bwd_tc"),
                                      "algorithmic": f"{MLP_FLOP_TRAIN} FLOP/sample (x3 bf16 MMAs executed)"},
        "k_adam": {"bound": "hbm", "achieved": adam_gbs, "peak": hbm, "unit": "GB/s", "frac": adam_gbs / hbm,
                   "traffic": traffic.get("k_adam"), "algorithmic": f"32 B/param x {n_par}"}}
    roofline_encode = {"encode_fwd": {"achieved": enc_fwd_gbs, "peak": hbm, "unit": "GB/s",
                                      "frac": enc_fwd_gbs / hbm,
                                      "bytes": f"{ENCODE_BYTES_PER_SAMPLE} B/sample x {samples_rank}"},
                       "encode_bwd": {"achieved": enc_bwd_gbs, "peak": hbm, "unit": "GB/s",
                                      "frac": enc_bwd_gbs / hbm,
                                      "bytes": f"{2 * ENCODE_BYTES_PER_SAMPLE} B/sample (atomic RMW)"},
                       "peak_kind": peak_kind}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        o, d, gt, _ = batches_host[0]
        cpu, why = cpu_reference(cfg, o, d, gt, args.cpu_rays, 1, 0, stages=not args.no_cpu_stages)
        if cpu is None:
            cpu = {"value": None, "unit": "rays/s", "cores": 0, "kind": "reference", "sample": why}
        else:
            cpu.pop("ms_per_step", None)
            cpu_stages = cpu.pop("stages", None)
            if cpu_stages and "unavailable" not in cpu_stages:
                # the same stages on the GPU, from this run's per-stage device times
                ms = lambda *k: sum(st[x] for x in k) / 1000.0
                cpu_stages["gpu_same_stages"] = {
                    "segment_march_rays_per_s": B / ms("segment", "march"),
                    "encode_samples_per_s": samples_rank / ms("encode_fwd"),
                    "field_fwd_samples_per_s": samples_rank / ms("encode_fwd", "mlp_fwd"),
                    "field_bwd_samples_per_s": samples_rank / ms("mlp_bwd", "encode_bwd"),
                    "adam_params_per_s": n_par / ms("adam")}
            cpu["stages"] = cpu_stages

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
                "data": "synthetic (random-init grids, drift-generator rays)",
                "config": {"workload": wl.name, "note": wl.note, "global_batch_rays": B,
                           "partitions": cfg.kx * cfg.ky, "tiling": [cfg.kx, cfg.ky],
                           "grid": {"L": 16, "F": 2, "T_log2": args.table_log2, "N0": 16, "Nmax": 2048},
                           "samples_per_step_rank0": samples_rank, "items_rank0": items_rank,
                           "l2": "working set > L2 (hash tables 1 GiB+/partition, sample buffers); "
                                 "3 distinct ray batches cycled",
                           "parallelism": f"partition-parallel x{world}"},
                "render_rays_per_s": render_value, "render_ms": rms,
                "encode_gbs": enc_fwd_gbs, "exchange_bytes_rank0": bytes_sent,
                "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
                "roofline": roof, "roofline_kernels": roofline_kernels, "roofline_encode": roofline_encode,
                "cpu_baseline": cpu}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
