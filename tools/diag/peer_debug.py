"""Two ranks on one GPU, host vs peer backend: item records and renders side by side
(diagnostic for dg_comm_init_peer)."""
import os
import socket
import sys

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def rank_main(rank, port, backend, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from tests import test_gpu_multirank as T
    from tests.helpers import app_rows, inject
    from paper_2405_04416_b200 import dg
    cfg = T._cfg(0)
    ctx = dg.Context(cfg, device=0, rank=rank, world=2)
    if backend == "peer":
        ctx.comm_init_peer(T._gloo_allgather)
    else:
        ctx.comm_init_host(T._gloo_alltoallv)
    inject(cfg, None, [T._LocalOnly(ctx)], occupancy_fraction=0.6)
    ctx.set_appearance(app_rows(1).astype(np.float32))
    o, d, gt, img = T._rays()
    lo, hi = rank * T.N // 2, (rank + 1) * T.N // 2
    app = app_rows(1)[0].astype(np.float32)
    rgb, Tr, depth = ctx.render(o[lo:hi], d[lo:hi], app, first_ray_id=lo)
    res = {"rgb": rgb, "T": Tr}
    for g in ctx.local:
        rid, order, te, tx, ns = ctx.last_item_data(g)
        res[f"rid{g}"], res[f"te{g}"], res[f"ns{g}"] = rid, te, ns
    np.savez(f"{out}_{backend}_{rank}.npz", **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    out = os.path.join(ROOT, "gpurun_out", "peerdbg")
    for backend in ("host", "peer"):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        ctx = mp.get_context("spawn")
        ps = [ctx.Process(target=rank_main, args=(r, port, backend, out)) for r in range(2)]
        [p.start() for p in ps]
        [p.join(300) for p in ps]
    for r in range(2):
        a = np.load(f"{out}_host_{r}.npz")
        b = np.load(f"{out}_peer_{r}.npz")
        for k in a.files:
            x, y = a[k], b[k]
            same = x.shape == y.shape and np.array_equal(x, y)
            print(r, k, x.shape, y.shape, "equal" if same else
                  f"DIFF max {np.abs(x.astype(float) - y.astype(float)).max() if x.shape == y.shape else 'shape'}")
            if not same and x.shape == y.shape and x.ndim == 1:
                bad = np.nonzero(x != y)[0]
                print("   first bad", bad[:10], x[bad[:5]], y[bad[:5]])
