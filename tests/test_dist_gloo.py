"""The N>1 (sharded) path on CPU with torch.distributed gloo, world_size 2/4.

Each rank owns one 2^M shard (numpy) and executes the PRODUCT's plan for
its rank (qsim_plan_json): pass / phase / perm ops with the rank bits in the
predicate, and every K-pair remap exchanged with gloo send/recv along the
routing the NCCL transport uses (qsim_exchange_peers).  Marginals
are reduced like qsim_probabilities across ranks (all_gather + fixed-order
sum).  The gathered state must equal the oracle's.
"""
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _apply(shard, full, code, t, cm, cv, m):
    if code == 6:
        return
    sel = (full & cm) == cv
    if code in (3, 5):
        shard[sel] *= complex(m[0], m[1])
        return
    tb = 1 << t
    i0 = np.nonzero(sel & ((full & tb) == 0))[0]
    i1 = i0 | tb
    x, y = shard[i0].copy(), shard[i1].copy()
    if code == 2:
        shard[i0], shard[i1] = y, x
        return
    u = [complex(m[0], m[1]), complex(m[2], m[3]), complex(m[4], m[5]), complex(m[6], m[7])]
    shard[i0] = u[0] * x + u[1] * y
    shard[i1] = u[2] * x + u[3] * y


def _chunk_index(M, lpos, v):
    """local indices whose bits lpos[i] equal bit i of v, ordered by the other bits"""
    idx = np.arange(1 << M, dtype=np.int64)
    sel = np.ones(1 << M, dtype=bool)
    for i, p in enumerate(lpos):
        sel &= ((idx >> p) & 1) == ((v >> i) & 1)
    return idx[sel]


def _worker(rank, world, port, case, out_q, policy=None):
    import torch
    import torch.distributed as dist
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_quant_ph_0608239_b200 as P
        from tests.plan_exec import _apply_u4, _store_remap
        n, init, gates, qs = case()
        plan = json.loads(P.plan_json(n, world, gates, policy=policy))
        G = (world - 1).bit_length()
        M = n - G
        phys0 = plan["initial_phys_of"]
        shard = np.zeros(1 << M, dtype=np.complex128)
        p0 = sum(((init >> q) & 1) << phys0[q] for q in range(n))
        if p0 >> M == rank:
            shard[p0 & ((1 << M) - 1)] = 1.0
        full = (np.int64(rank) << M) | np.arange(1 << M, dtype=np.int64)
        n_ex = 0
        for st in plan["plan"]["steps"]:
            ty = st["type"]
            if ty == "pass":
                for op in st["ops"]:
                    if op["code"] == 7:  # fused 4x4 block on two local bits
                        _apply_u4(shard, np.arange(1 << M, dtype=np.int64), op["t"], op["t2"], op["m"])
                    elif op["code"] not in (4, 6, 8):
                        _apply(shard, full, op["code"], op["t"], op["cm"], op["cv"], op["m"])
                shard = _store_remap(shard, np.arange(1 << M, dtype=np.int64), st["tp"], st["tp_out"])
            elif ty == "generic":
                _apply(shard, full, st["code"], st["t"], st["cm"], st["cv"], st["m"])
            elif ty == "phase":
                _apply(shard, full, 3, -1, st["cm"], st["cv"], st["m"])
            elif ty == "permrun":
                loc = np.arange(1 << M, dtype=np.int64)
                for gid, cm in zip(st["gates"], st["cms"]):
                    w = np.zeros(1 << M, dtype=np.int64)
                    for b, p in enumerate(st["targets"]):
                        w |= ((loc >> p) & 1) << b
                    pw = np.asarray(gates[gid].perm, dtype=np.int64)[w]
                    dest = loc.copy()
                    for b, p in enumerate(st["targets"]):
                        dest = (dest & ~(1 << p)) | (((pw >> b) & 1) << p)
                    sel = (full & cm) == cm
                    new = shard.copy()
                    new[dest[sel]] = shard[sel]
                    shard = new
            elif ty == "perm":
                g = gates[st["gate"]]
                T, cm = st["targets"], st["cm"]
                w = np.zeros(1 << M, dtype=np.int64)
                for b, p in enumerate(T):
                    w |= ((np.arange(1 << M, dtype=np.int64) >> p) & 1) << b
                pw = np.asarray(g.perm, dtype=np.int64)[w]
                dest = np.arange(1 << M, dtype=np.int64)
                for b, p in enumerate(T):
                    dest = (dest & ~(1 << p)) | (((pw >> b) & 1) << p)
                sel = (full & cm) == cm
                new = shard.copy()
                new[dest[sel]] = shard[sel]
                shard = new
            elif ty == "exchange":
                lpos, gpos = st["lpos"], st["gpos"]
                peers, selfv = P.exchange_peers(n, world, rank, gpos)
                reqs, bufs = [], {}
                for v in range(1 << len(lpos)):
                    if v == selfv:
                        continue
                    ci = _chunk_index(M, lpos, v)
                    send = torch.from_numpy(shard[ci].view(np.float64).copy())
                    recv = torch.empty_like(send)
                    reqs.append(dist.isend(send, peers[v]))
                    reqs.append(dist.irecv(recv, peers[v]))
                    bufs[v] = (ci, recv, send)
                for r in reqs:
                    r.wait()
                for v, (ci, recv, _) in bufs.items():
                    shard[ci] = recv.numpy().view(np.complex128)
                n_ex += 1
            elif ty == "pairwise":
                gb = 1 << (st["t"] - M)
                peer = rank ^ gb
                lm = (1 << M) - 1
                if ((rank << M) & st["cm"] & ~lm) == (st["cv"] & ~lm):
                    send = torch.from_numpy(shard.view(np.float64).copy())
                    recv = torch.empty_like(send)
                    reqs = [dist.isend(send, peer), dist.irecv(recv, peer)]
                    for r_ in reqs:
                        r_.wait()
                    other = recv.numpy().view(np.complex128)
                    m = st["m"]
                    u = [complex(m[0], m[1]), complex(m[2], m[3]), complex(m[4], m[5]), complex(m[6], m[7])]
                    if st["code"] == 2:
                        u = [0, 1, 1, 0]
                    sel = (np.arange(1 << M) & st["cm"] & lm) == (st["cv"] & lm)
                    if rank & gb:
                        shard[sel] = u[2] * other[sel] + u[3] * shard[sel]
                    else:
                        shard[sel] = u[0] * shard[sel] + u[1] * other[sel]
                n_ex += 1
        # gather the state (logical order) and reduce a marginal like qsim_probabilities
        allsh = [torch.empty(2 << M, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allsh, torch.from_numpy(shard.view(np.float64).copy()))
        phys = np.concatenate([a.numpy().view(np.complex128) for a in allsh])
        fin = plan["plan"]["final_phys_of"]
        x = np.arange(1 << n, dtype=np.int64)
        pidx = np.zeros_like(x)
        for q in range(n):
            pidx |= ((x >> q) & 1) << fin[q]
        logical = phys[pidx]
        beta = np.zeros(1 << M, dtype=np.int64)
        for b, q in enumerate(qs):
            beta |= ((full >> fin[q]) & 1) << b
        part = np.bincount(beta, weights=np.abs(shard) ** 2, minlength=1 << len(qs))
        parts = [torch.empty(1 << len(qs), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(part))
        prob = np.zeros(1 << len(qs))
        for r in range(world):  # fixed rank order
            prob += parts[r].numpy()
        if rank == 0:
            out_q.put((logical, prob, n_ex))
    finally:
        dist.destroy_process_group()


def _case_brickwork():
    from workloads import circuits as C
    return 13, 5, C.random_brickwork(13, 5, seed=21), [12, 0, 7]


def _case_chain4():
    from workloads import circuits as C
    return 14, 0, C.random_chain(14, 2, seed=4, sweep=True), [13, 12, 1]


def _case_shor():
    from workloads import circuits as C
    w = C.shor_order_finding(35, 3, 8, 6)
    return w.n, w.init, w.gates, list(range(8))


def _case_qft():
    from workloads import circuits as C
    w = C.qft_basis(13, 777)
    return 13, w.init, w.gates, [12, 11]


@pytest.mark.parametrize("world,case,policy", [(2, _case_brickwork, None), (2, _case_shor, None), (2, _case_qft, None),
                                               (4, _case_chain4, None), (2, _case_brickwork, "pairwise"),
                                               (4, _case_chain4, "pairwise")])
def test_sharded_path_gloo(oracle_mod, world, case, policy):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, policy)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        logical, prob, n_ex = q.get(timeout=120)
    except Exception:
        for p in procs:
            p.kill()
        raise
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, init, gates, qs = case()
    o = oracle_mod.Oracle(n)
    o.init_basis(init)
    o.run(gates)
    assert np.max(np.abs(logical - o.amplitudes())) <= 1e-12
    assert np.max(np.abs(prob - o.probabilities(qs))) <= 1e-13
    assert n_ex >= 1
