"""Multi-rank exchange protocol on CPU (gloo, world size 2 and 3): the host-side layouts of
both per-step exchanges (dg_plan_dispatch / dg_plan_partials, exchange_plan.cpp) are driven
with synthetic ray schedules, the exchanges are simulated with torch.distributed all-to-all,
and every rank checks it received exactly the reference's item set in ray order
(Worker::handle_training_batch dispatch, worker.cpp:251-313) and, per stream (q -> p), the
partials of exactly the rays through both q and p in ray order (PartialScatter,
worker.cpp:314-360).  No GPU involved: the planner is host code in libdg_b200.so."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REC, PART = 72, 24  # RayRec / PartialRec bytes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _schedules(n, P, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        k = int(rng.integers(0, min(P, 4) + 1))  # 0 = dropped ray (misses every region)
        out.append(list(rng.permutation(P)[:k]))
    return out


def _a2a(blocks_per_dst, world):
    """All-to-all of int64 row blocks; returns the received blocks in source-rank order."""
    send_sizes = [len(b) for b in blocks_per_dst]
    sizes = torch.tensor(send_sizes, dtype=torch.int64)
    recv_sizes = torch.empty(world, dtype=torch.int64)
    dist.all_to_all_single(recv_sizes, sizes)
    width = 3
    send = torch.from_numpy(np.concatenate([np.asarray(b, np.int64).reshape(-1, width) for b in blocks_per_dst])
                            if sum(send_sizes) else np.zeros((0, width), np.int64)).reshape(-1)
    recv = torch.empty(int(recv_sizes.sum()) * width, dtype=torch.int64)
    dist.all_to_all_single(recv, send, [int(r) * width for r in recv_sizes], [s * width for s in send_sizes])
    out, off = [], 0
    rv = recv.numpy().reshape(-1, width)
    for r in range(world):
        out.append(rv[off:off + int(recv_sizes[r])])
        off += int(recv_sizes[r])
    return out


def _worker(rank, world, port, P, n, seed, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2405_04416_b200 import dg
        sched = _schedules(n, P, seed)
        lo, hi = rank * n // world, (rank + 1) * n // world  # contiguous home shard
        local = [p for p in range(P) if p % world == rank]
        # ---- exchange 1: rays -> owners ----
        send_cnt = np.zeros(P, np.uint64)
        for i in range(lo, hi):
            for p in sched[i]:
                send_cnt[p] += 1
        allc = [torch.zeros(P, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, torch.from_numpy(send_cnt.astype(np.int64)))
        cnt_recv = np.stack([c.numpy() for c in allc]).astype(np.uint64)
        sb, rb, item_off, bsrc, bdst = dg.plan_dispatch(rank, world, P, send_cnt, cnt_recv)
        # send buffer [dest r][partition on r (ascending)][ray]
        blocks = []
        for r in range(world):
            rows = [(i, p, 0) for p in range(P) if p % world == r for i in range(lo, hi) if p in sched[i]]
            assert len(rows) * REC == int(sb[r])
            blocks.append(rows)
        got = _a2a(blocks, world)
        for r in range(world):
            assert len(got[r]) * REC == int(rb[r]), (rank, r)
        recv = np.concatenate(got) if sum(len(g) for g in got) else np.zeros((0, 3), np.int64)
        items = np.zeros_like(recv)
        nl = len(local)
        for b in range(world * nl):  # block permutation recv [src][lp] -> items [lp][src]
            r, lp = divmod(b, nl)
            c = int(cnt_recv[r][local[lp]])
            items[int(bdst[b]):int(bdst[b]) + c] = recv[int(bsrc[b]):int(bsrc[b]) + c]
        for lp, p in enumerate(local):
            want = [i for i in range(n) if p in sched[i]]
            have = items[int(item_off[lp]):int(item_off[lp + 1])]
            assert list(have[:, 0]) == want, (rank, p)
            assert (have[:, 1] == p).all()
        # ---- exchange 2: partials among owners ----
        pair = np.zeros((nl, P), np.uint32)
        for lp, p in enumerate(local):
            for i in items[int(item_off[lp]):int(item_off[lp + 1]), 0]:
                for q in sched[i]:
                    if q != p:
                        pair[lp, q] += 1
        so, ro, psb, prb = dg.plan_partials(rank, world, P, pair)
        total = int(sum(psb)) // PART
        sendbuf = np.full((total, 3), -1, np.int64)
        for lq, q in enumerate(local):
            k = {}
            for i in items[int(item_off[lq]):int(item_off[lq + 1]), 0]:  # ray order
                for p in sched[i]:
                    if p != q:
                        sendbuf[int(so[q, p]) + k.get(p, 0)] = (i, q, p)
                        k[p] = k.get(p, 0) + 1
        assert (sendbuf[:, 0] >= 0).all()
        blocks, off = [], 0
        for r in range(world):
            c = int(psb[r]) // PART
            blocks.append(sendbuf[off:off + c])
            off += c
        got = _a2a(blocks, world)
        for r in range(world):
            assert len(got[r]) * PART == int(prb[r]), (rank, r)
        recv = np.concatenate(got) if sum(len(g) for g in got) else np.zeros((0, 3), np.int64)
        for p in local:
            for q in range(P):
                if q == p:
                    continue
                want = [i for i in range(n) if p in sched[i] and q in sched[i]]
                o = int(ro[q, p])
                have = recv[o:o + len(want)]
                assert list(have[:, 0]) == want, (rank, q, p)
                assert (have[:, 1] == q).all() and (have[:, 2] == p).all()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported by the parent
        import traceback
        errq.put((rank, traceback.format_exc()))
        raise


@pytest.mark.parametrize("world,P", [(2, 2), (2, 5), (3, 7)])
def test_exchange_plans_multirank_gloo(world, P):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, 240, 11 + P, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_plan_single_rank_aliases():
    """world = 1: every stream is local, send and recv layouts coincide (the runtime aliases)."""
    from paper_2405_04416_b200 import dg
    P = 4
    pair = np.array([[0, 3, 1, 0], [3, 0, 2, 2], [1, 2, 0, 5], [0, 2, 5, 0]], np.uint32)
    so, ro, sb, rb = dg.plan_partials(0, 1, P, pair)
    assert (so == ro).all() and int(sb[0]) == int(rb[0]) == int(pair.sum()) * PART
