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


def profile_traffic(workload):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the hot kernels
    from the committed ncu --set full capture of this workload (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        w = tj["workloads"][workload]
        out = {k: v["dram_bytes_per_launch"] for k, v in w["kernels"].items()}
        out["_source"] = w.get("source", "")
        return out
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
    bounded sample of `rays` rays of the same workload (its K worker threads + driver)."""
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
                      f"workload (K={cfg.kx * cfg.ky} worker thread(s); reference init {init_s:.1f}s excluded)",
            "ms_per_step": 1000 * sec / len(times), "stages": stage}, None


REF_PARTITION_BYTES = 11.5e9  # one reference partition (Worker) at T = 2^24 (tools/diag/ref_rss.py: 10.7 GB)


def no_update_steps(first, n, interval=16):
    """n step ids >= first whose step does not run Worker::update_occupancy."""
    out, s = [], first
    while len(out) < n:
        if (s + 1) % interval:
            out.append(s)
        s += 1
    return out


def cpu_reference_replicas(cfg, rays_per_partition, steps, warmup, generator):
    """The reference on every host thread it can use.  DistributedRun parallelises only across
    partitions (one worker thread each), so the host runs independent replicas of the whole
    K-partition DistributedRun, each on its own slice of the workload (rays_per_partition x K
    rays per step), in lock step on one thread group (ref_harness.cpp refh_time_replicas), over
    the same step indices as the GPU arm: W warm-up steps 0..W-1, then K timed steps.  The
    replica count is capped by host memory.  Also measured: the marginal (Adam-excluded) rate
    from one replica at two batch sizes, since the dense Adam over every parameter is a fixed
    per-step cost that does not scale with rays (worker.cpp:524-547)."""
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
    K = cfg.kx * cfg.ky
    per_part = REF_PARTITION_BYTES * (2.0 ** (cfg.fine_table_log2 - 24)) if cfg.fine_table_log2 >= 20 else 1e9
    n_rep = int(max(1, min(nproc // K if nproc >= K else 1, (0.45 * avail) // (per_part * K))))
    rays = rays_per_partition * K
    o, d, gt, _ = workloads.make_rays(cfg, n_rep * rays, generator, seed=1)
    app = workloads.appearance_rows(cfg.appearance_dim, 1)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(n_rep) as ex:  # refh_create runs without the GIL
        runs = list(ex.map(lambda _: RefRun(cfg, app), range(n_rep)))
    init_s = time.perf_counter() - t0
    lib = ref_lib()
    o, d, gt = (np.ascontiguousarray(x, np.float64) for x in (o, d, gt))
    P = C.c_void_p

    def run_steps(handles, n_runs, nrays, nsteps, first):
        return lib.refh_time_replicas(handles, n_runs, o.ctypes.data_as(P), d.ctypes.data_as(P),
                                      gt.ctypes.data_as(P), nrays, nsteps, first)

    handles = (C.c_void_p * n_rep)(*[r.h for r in runs])
    if warmup and run_steps(handles, n_rep, rays, warmup, 0) < 0:
        return None, lib.refh_last_error().decode()
    sec = run_steps(handles, n_rep, rays, steps, warmup)
    if sec < 0:
        return None, lib.refh_last_error().decode()
    # marginal cost per ray: one replica, steps without an occupancy update, two batch sizes
    one = (C.c_void_p * 1)(runs[0].h)
    ids = no_update_steps(warmup + steps, 2)
    small = max(1, rays // 4)
    t_big = run_steps(one, 1, rays, 1, ids[0])
    t_small = run_steps(one, 1, small, 1, ids[1])
    marginal = None
    if t_big > 0 and t_small > 0 and t_big > t_small:
        per_ray = (t_big - t_small) / (rays - small)
        marginal = {"value": n_rep / per_ray, "unit": "rays/s",
                    "fixed_ms_per_step": 1000 * (t_big - per_ray * rays),
                    "method": f"one replica, DistributedRun::training_step at {rays} and {small} rays "
                              f"(steps {ids[0]}, {ids[1]}): {n_rep} replicas / marginal s per ray; the "
                              "fixed part is the dense Adam + zeroing over every parameter"}
    del runs
    value = n_rep * rays * steps / sec
    return {"value": value, "unit": "rays/s", "cores": n_rep * K, "kind": "reference",
            "sample": f"{n_rep} replica(s) of the reference DistributedRun with K={K} worker thread(s) "
                      f"each (+ its driver thread; the reference parallelises only across partitions), "
                      f"{rays} rays/step each ({rays_per_partition} per partition), {warmup} warm-up + "
                      f"{steps} timed lock-step steps (step ids {warmup}..{warmup + steps - 1}); "
                      f"{nproc}-thread host ({model}); init {init_s:.1f}s excluded",
            "ms_per_step": 1000 * sec / steps, "adam_excluded": marginal, "warmup_run": warmup}, None


def workload_config(wl, world, table_log2, mode="train"):
    cfg = wl.cfg
    return {"workload": wl.name, "mode": mode, "note": wl.note, "global_batch_rays": wl.n_rays,
            "partitions": cfg.kx * cfg.ky, "tiling": [cfg.kx, cfg.ky],
            "grid": {"L": cfg.grid_levels, "F": cfg.grid_features, "T_log2": cfg.fine_table_log2,
                     "N0": cfg.base_resolution, "Nmax": cfg.max_resolution},
            "march_step_divisor": cfg.march_step_divisor, "generator": wl.generator,
            "l2": "inputs larger than L2 (hash tables 1 GiB+/partition, ~4 GB of per-sample "
                  "buffers per step); 3 distinct ray batches cycled",
            "parallelism": f"partition-parallel x{world} (partition p on rank p % {world})"}


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from paper_2405_04416_b200 import workloads
    n = max(world, args.gpus)
    wl = workloads.weak(n, rays_per_gpu=args.rays_per_gpu, table_log2=args.table_log2)
    res, why = cpu_reference_replicas(wl.cfg, args.ref_rays, args.steps, args.warmup, wl.generator)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": why}))
        return 0
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": "rays/s",
            "n_gpus": n, "steps": args.steps, "warmup": res["warmup_run"],
            "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference init, drift-generator rays)",
            "config": workload_config(wl, n, args.table_log2),
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "adam_excluded": res["adam_excluded"],
            "e2e": {"value": res["value"], "unit": "rays/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: run N ranks under torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ our arm
def make_batches(wl, lo, hi, nb):
    from paper_2405_04416_b200 import workloads
    out = []
    for k in range(nb):
        o, d, gt, img = workloads.make_rays(wl.cfg, wl.n_rays, wl.generator, seed=1 + k)
        out.append((o[lo:hi], d[lo:hi], gt[lo:hi], img[lo:hi]))
    return out


def device_batches(batches_host, lo, abi, torch):
    dev = []
    for (o, d, gt, img) in batches_host:
        t = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (o, d, gt, img.astype(np.int32))]
        b = abi.RayBatch()
        b.origin, b.dir, b.color_gt, b.image_id = (t[0].data_ptr(), t[1].data_ptr(),
                                                   t[2].data_ptr(), t[3].data_ptr())
        b.n, b.first_ray_id, b.mem = len(o), lo, abi.DG_MEM_DEVICE
        dev.append((b, t))
    return dev


def pinned_batches(batches_host, lo, abi, torch):
    out = []
    for (o, d, gt, img) in batches_host:
        t = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (o, d, gt, img.astype(np.int32))]
        b = abi.RayBatch()
        b.origin, b.dir, b.color_gt, b.image_id = (t[0].data_ptr(), t[1].data_ptr(),
                                                   t[2].data_ptr(), t[3].data_ptr())
        b.n, b.first_ray_id, b.mem = len(o), lo, abi.DG_MEM_HOST
        out.append((b, t))
    return out


class Runner:
    """One context on this rank plus the timing helpers (CUDA events on the context's stream,
    barrier + synchronize on both sides, max over ranks)."""

    def __init__(self, wl, rank, world, local, comm, torch, dist):
        from paper_2405_04416_b200 import abi, dg, workloads
        self.abi, self.dg, self.torch, self.dist = abi, dg, torch, dist
        self.wl, self.rank, self.world = wl, rank, world
        cfg = wl.cfg
        self.ctx = dg.Context(cfg, device=local, rank=rank, world=world)
        if world > 1:
            uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                uid.copy_(torch.tensor(list(dg.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, 0)
            if comm == "peer":  # pack kernels write the owners' buffers over CUDA IPC
                gloo = dist.new_group(backend="gloo")

                def allgather(blob):
                    out = [None] * world
                    dist.all_gather_object(out, blob, group=gloo)
                    return out

                self.ctx.comm_init_peer(allgather)
            else:
                self.ctx.comm_init_nccl(bytes(uid.cpu().tolist()))
        for g in self.ctx.local:
            self.ctx.init_fast(g, seed=1)
        self.ctx.set_appearance(workloads.appearance_rows(cfg.appearance_dim, 1))
        sptr = C.c_void_p()
        dg.lib().dg_get_stream(self.ctx.h, C.byref(sptr))
        self.stream = torch.cuda.ExternalStream(sptr.value)
        self.stats = abi.StepStats()
        self.samples = 0
        self.h2d = self.d2h = 0  # host <-> device bytes of the steps run (copies through the ABI)
        self.shard = wl.n_rays // world
        self.lo = rank * self.shard

    def step(self, i, batches):
        rc = self.ctx.train_step_raw(batches[i % len(batches)][0], i, self.stats)
        if rc != 0:
            raise self.dg.DGError(rc, self.dg.lib().dg_last_error().decode())
        self.samples += int(self.stats.samples)
        self.h2d += int(self.stats.h2d_bytes)
        self.d2h += int(self.stats.d2h_bytes)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, v):
        if self.world > 1:
            t = self.torch.tensor([float(v)], device="cuda")
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
            v = float(t.item())
        return v

    def sum_over_ranks(self, v):
        if self.world > 1:
            t = self.torch.tensor([float(v)], device="cuda", dtype=self.torch.float64)
            self.dist.all_reduce(t)
            v = float(t.item())
        return v

    def timed(self, fn, n, first):
        torch = self.torch
        self.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        for i in range(n):
            fn(first + i)
        self.ctx.fence()  # the last step's Adam (side stream) inside the timed region
        e1.record(self.stream)
        e1.synchronize()
        self.barrier()
        return self.max_over_ranks(e0.elapsed_time(e1))

    def render_rate(self, batches, steps, warmup=3):
        torch, abi = self.torch, self.abi
        m = abi.Merged()
        out = [torch.empty(x, device="cuda") for x in ((self.shard, 3), (self.shard,), (self.shard,))]
        m.rgb, m.transmittance, m.depth, m.mem = (out[0].data_ptr(), out[1].data_ptr(),
                                                   out[2].data_ptr(), abi.DG_MEM_DEVICE)
        from paper_2405_04416_b200 import workloads
        app = np.ascontiguousarray(workloads.appearance_rows(self.wl.cfg.appearance_dim, 1)[0], dtype=np.float32)

        def render(i):
            rc = self.ctx.render_raw(batches[i % len(batches)][0], app, m)
            if rc != 0:
                raise self.dg.DGError(rc, self.dg.lib().dg_last_error().decode())

        for i in range(max(warmup, 1)):
            render(i)
        l0 = self.ctx.kernel_launches()
        rms = self.timed(render, steps, 0) / steps
        return self.wl.n_rays / (rms / 1000.0), rms, self.ctx.kernel_launches() - l0

    def close(self):
        self.ctx.close()


def extra_workloads(rank, world, local, args, torch, dist):
    """Driver-visible lines for the other BASELINE configs on the GPUs of this run: C1 (train
    + render, one partition, T=2^19; world = 1 only) and the C5 render-only sweep point (8
    partitions, worst-case 5-segment rays; partition p on rank p % world)."""
    from paper_2405_04416_b200 import workloads
    out = {}
    todo = (["C1"] if world == 1 else []) + ["C5"]
    for name in todo:
        wl = workloads.by_name(name)
        r = Runner(wl, rank, world, local, args.comm, torch, dist)
        hb = make_batches(wl, r.lo, r.lo + r.shard, 2)
        dev = device_batches(hb, r.lo, r.abi, torch)
        ent = {"config": workload_config(wl, world, wl.cfg.fine_table_log2,
                                         "train+render" if name == "C1" else "render")}
        if name == "C1":
            for i in range(3):
                r.step(i, dev)
            r.samples = 0
            ms = r.timed(lambda i: r.step(i, dev), 4, 3) / 4
            ent["train_rays_per_s"] = wl.n_rays / (ms / 1000.0)
            ent["train_ms_per_step"] = ms
            ent["samples_per_step"] = r.sum_over_ranks(r.samples) / 4
        rv, rms, _ = r.render_rate(dev, 4)
        ent["render_rays_per_s"] = rv
        ent["render_ms"] = rms
        out[name] = ent
        r.close()
        del r, dev
        torch.cuda.empty_cache()
    return out


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
    ap.add_argument("--no-extra", action="store_true", help="skip the C1 / C5 render lines")
    ap.add_argument("--workload", default="weak", choices=["weak", "C1", "C2", "C3", "C4", "C5"],
                    help="weak: the C4 weak-scaling point (default); C1..C4: a BASELINE config whole "
                         "(training); C5: the render-only worst case")
    ap.add_argument("--comm", default="peer", choices=["nccl", "peer"],
                    help="exchange backend for N > 1: peer-memory pack kernels (the transfer fused "
                         "into the pack kernels over CUDA-IPC / NVLink, default) or NCCL all-to-all-v")
    ap.add_argument("--no-cpu-stages", action="store_true", help="skip the all-core stage baseline")
    ap.add_argument("--ref-rays", type=int, default=4096,
                    help="rays per partition per step of each reference replica (SURVEY 8d (i): 4,096)")
    ap.add_argument("--cpu-rays", type=int, default=2048, help="rays of the cpu_baseline sample (~10 s)")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    args = ap.parse_args()
    rank, world, local = env_rank()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    from paper_2405_04416_b200 import workloads

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    render_only = args.workload == "C5"
    if args.workload == "weak":
        wl = workloads.weak(world, rays_per_gpu=args.rays_per_gpu, table_log2=args.table_log2)
    else:  # a BASELINE config as a whole on `world` GPUs (partition p on rank p % world)
        wl = workloads.by_name(args.workload)
        args.no_cpu = args.no_extra = True
    cfg = wl.cfg
    B = wl.n_rays
    r = Runner(wl, rank, world, local, args.comm, torch, dist)
    ctx = r.ctx
    NB = 1 if args.profile else 3  # distinct batches cycled over the steps
    batches_host = make_batches(wl, r.lo, r.lo + r.shard, NB)
    dev = device_batches(batches_host, r.lo, r.abi, torch)
    hbm, tensor_peak, peak_kind = peaks()
    config = workload_config(wl, world, cfg.fine_table_log2, "render" if render_only else "train")

    if render_only:
        with ClockSampler(local) as clk:
            rv, rms, launches = r.render_rate(dev, max(args.steps, 1), max(args.warmup, 1))
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": rv, "unit": "rays/s", "n_gpus": world,
                              "steps": max(args.steps, 1), "warmup": max(args.warmup, 1),
                              "clocks": clk.summary(), "ms_per_step": rms,
                              "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                              "dtype": "fp32", "data": "synthetic (random-init grids, corner rays)",
                              "config": config, "gpu_launches": int(launches), "e2e": None,
                              "roofline": None, "cpu_baseline": None}))
        if world > 1:
            dist.destroy_process_group()
        return 0

    for i in range(args.warmup):
        r.step(i, dev)
    ctx.snapshot()  # the state the timed window starts from (replayed by the e2e pass)
    r.samples = 0
    launches0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        ms = r.timed(lambda i: r.step(i, dev), args.steps, args.warmup)
    launches = ctx.kernel_launches() - launches0
    ms_per_step = ms / args.steps
    value = B / (ms_per_step / 1000.0)
    samples_step = r.sum_over_ranks(r.samples) / args.steps  # mean over the window, all ranks
    samples_rank = r.samples / args.steps
    items_rank = int(r.stats.items)
    bytes_sent = int(r.stats.bytes_sent)

    # per-stage device times of one more step (events on the step stream)
    ctx.enable_stage_timing(True)
    r.step(args.warmup + args.steps, dev)
    st = ctx.stage_times()
    ctx.enable_stage_timing(False)
    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_per_step, "stages_ms": st}))
        if world > 1:
            dist.destroy_process_group()
        return 0

    # end-to-end through the C ABI with pinned host buffers, over the same step indices from
    # the same state (dg_state_snapshot): e2e - value = the host <-> device copies
    e2e = None
    if not args.no_e2e:
        pinned = pinned_batches(batches_host, r.lo, r.abi, torch)
        ctx.snapshot(restore=True)
        r.step(args.warmup, pinned)  # first host-batch step allocates the staging buffers
        ctx.snapshot(restore=True)
        r.samples = 0
        r.h2d = r.d2h = 0
        ems = r.timed(lambda i: r.step(i, pinned), args.steps, args.warmup)
        # mean over the window: the ray batch every step, plus the occupancy update's sample
        # stream (uploaded once per update, ahead of it) in the window's update step
        e2e = {"value": B / (ems / args.steps / 1000.0), "unit": "rays/s",
               "h2d_bytes_per_step": r.h2d // args.steps, "d2h_bytes_per_step": r.d2h // args.steps,
               "batch_h2d_bytes_per_step": int(B // world * (48 + 12 + 4)),
               "ms_per_step": ems / args.steps, "same_steps_and_state_as_value": True,
               "samples_per_step": r.sum_over_ranks(r.samples) / args.steps}

    # render throughput (evaluate_rays through the same kernels)
    render_value, rms, _ = r.render_rate(dev, args.render_steps)

    # exchange efficiency (NVLink all-to-all bytes / time vs 900 GB/s per direction)
    exchange = None
    if world > 1:
        x1_ms = r.max_over_ranks(st["dispatch_exchange"])
        x2_ms = r.max_over_ranks(st["exchange"])
        mb = r.max_over_ranks(st["dispatch_mb"] + st["partial_mb"])
        gbs = mb * 1e6 / ((x1_ms + x2_ms) / 1e3) / 1e9 if x1_ms + x2_ms > 0 else None
        exchange = {"bytes_per_step_max_rank": mb * 1e6, "dispatch_ms": x1_ms, "partials_ms": x2_ms,
                    "achieved_gbs": gbs, "peak_gbs": 900.0, "frac": gbs / 900.0 if gbs else None,
                    "backend": args.comm,
                    "note": "bytes a rank sends to other ranks in both exchanges / the two exchanges' "
                            "device time (max over ranks), vs NVLink 5 per direction"}

    # roofline of the dominant kernel + every hot kernel against its own roof
    enc_bytes = samples_rank * ENCODE_BYTES_PER_SAMPLE
    stage_ms = {k: v for k, v in st.items()
                if k not in ("total", "dispatch_exchange", "dispatch_mb", "partial_mb")}
    dominant = max(stage_ms, key=stage_ms.get)
    enc_fwd_gbs = enc_bytes / (st["encode_fwd"] / 1e3) / 1e9 if st["encode_fwd"] > 0 else 0.0
    enc_bwd_gbs = 2 * enc_bytes / (st["encode_bwd"] / 1e3) / 1e9 if st["encode_bwd"] > 0 else 0.0
    mlp_tflops = samples_rank * MLP_FLOP_TRAIN / ((st["mlp_fwd"] + st["mlp_bwd"]) / 1e3) / 1e12
    traffic = profile_traffic(wl.name)
    if dominant in ("mlp_fwd", "mlp_bwd"):
        roof = {"kernel": "k_mlp_fwd_tc+k_mlp_bwd_tc_relu", "bound": "tensor", "achieved": mlp_tflops,
                "peak": tensor_peak, "unit": "TFLOP/s", "frac": mlp_tflops / tensor_peak,
                "traffic": traffic.get("k_mlp_bwd_tc_relu", traffic.get("k_mlp_bwd_tc")),
                "note": f"{MLP_FLOP_TRAIN} algorithmic FLOP/sample x {samples_rank:.0f} samples; peak = "
                        f"{peak_kind} sustained dense bf16"}
    else:
        ach = {"encode_fwd": enc_fwd_gbs, "encode_bwd": enc_bwd_gbs}.get(dominant, enc_fwd_gbs)
        kname = {"encode_fwd": "k_encode_fwd", "encode_bwd": "k_encode_bwd"}.get(dominant, dominant)
        roof = {"kernel": kname, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": traffic.get(kname),
                "note": "achieved = algorithmic bytes (SURVEY 8d: 1024 B/sample forward, 2048 B/sample "
                        "RMW backward) / the kernel's live CUDA-event time on the step stream; traffic = "
                        f"DRAM read+write bytes per launch from the ncu --set full capture of this "
                        f"workload (profiles/traffic.json, {traffic.get('_source', 'none')})"}
    roof["stage_ms"] = st
    n_par = sum(ctx.param_count(g) for g in ctx.local)
    adam_gbs = 32.0 * n_par / (st["adam"] / 1e3) / 1e9 if st["adam"] > 0 else 0.0
    roofline_kernels = {
        "k_encode_fwd": {"bound": "hbm", "achieved": enc_fwd_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": enc_fwd_gbs / hbm, "traffic": traffic.get("k_encode_fwd"),
                         "algorithmic": f"{ENCODE_BYTES_PER_SAMPLE} B/sample"},
        "k_encode_bwd": {"bound": "hbm (L2 atomics)", "achieved": enc_bwd_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": enc_bwd_gbs / hbm, "traffic": traffic.get("k_encode_bwd"),
                         "algorithmic": f"{2 * ENCODE_BYTES_PER_SAMPLE} B/sample (RMW)"},
        "k_mlp_fwd_tc+k_mlp_bwd_tc_relu": {"bound": "tensor", "achieved": mlp_tflops, "peak": tensor_peak,
                                           "unit": "TFLOP/s", "frac": mlp_tflops / tensor_peak,
                                           "traffic": traffic.get("k_mlp_bwd_tc_relu", traffic.get("k_mlp_bwd_tc")),
                                      "algorithmic": f"{MLP_FLOP_TRAIN} FLOP/sample (forward split-tf32, "
                                                     "backward split-bf16: 3 MMAs per product executed)"},
        "k_adam": {"bound": "hbm", "achieved": adam_gbs, "peak": hbm, "unit": "GB/s", "frac": adam_gbs / hbm,
                   "traffic": traffic.get("k_adam"), "algorithmic": f"32 B/param x {n_par}"}}

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
                ms_of = lambda *k: sum(st[x] for x in k) / 1000.0
                cpu_stages["gpu_same_stages"] = {
                    "segment_march_rays_per_s": B / ms_of("segment", "march"),
                    "encode_samples_per_s": samples_rank / ms_of("encode_fwd"),
                    "field_fwd_samples_per_s": samples_rank / ms_of("encode_fwd", "mlp_fwd"),
                    "field_bwd_samples_per_s": samples_rank / ms_of("mlp_bwd", "encode_bwd"),
                    "adam_params_per_s": n_par / ms_of("adam")}
            cpu["stages"] = cpu_stages
    r.close()
    del r, dev
    torch.cuda.empty_cache()
    extra = None
    if not args.no_extra:
        extra = extra_workloads(rank, world, local, args, torch, dist)

    if rank == 0:
        config.update({"samples_per_step": samples_step, "samples_per_step_rank0": samples_rank,
                       "items_rank0": items_rank,
                       "timed_steps": f"{args.warmup}..{args.warmup + args.steps - 1} (occupancy update "
                                      f"every 16 steps: after steps 15, 31, ...)"})
        line = {"metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
                "data": "synthetic (random-init grids, drift-generator rays)", "config": config,
                "render_rays_per_s": render_value, "render_ms": rms,
                "encode_gbs": enc_fwd_gbs, "exchange_bytes_rank0": bytes_sent, "exchange": exchange,
                "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
                "roofline": roof, "roofline_kernels": roofline_kernels, "peak_kind": peak_kind,
                "cpu_baseline": cpu, "workloads": extra}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
