"""World-size-2 CPU (gloo) coverage of the row-sharded schedule.

The NCCL path itself needs GPUs; here two processes run the SAME schedule as
paper_2212_02406_b200/csrc/sharded.cu with torch.distributed (gloo) standing in
for NCCL and numpy for the local DMMA GEMMs:
  * row blocks from the library's own nnb_partition_rows (16-row units),
  * ring all-gather in G-1 send/recv steps, partial products own block first
    then in ring order (K split by the ranks' row blocks),
  * eps from the per-rank Σ‖R_g‖² all-gathered and summed in rank order.
Checked against the single-process oracle chain and for bit-identical eps on
every rank (identical stop decisions)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2212_02406_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ring_allgather(full, row0, rows, me, G):
    """In-place ring all-gather of row blocks, same step order as ring_allgather()."""
    for q in range(1, G):
        send_blk, recv_blk = (me - q + 1) % G, (me - q) % G
        sbuf = torch.from_numpy(np.ascontiguousarray(full[row0[send_blk]:row0[send_blk] + rows[send_blk]]))
        rbuf = torch.empty((rows[recv_blk], full.shape[1]), dtype=torch.float64)
        reqs = [dist.isend(sbuf, (me + 1) % G), dist.irecv(rbuf, (me - 1) % G)]
        for r in reqs:
            r.wait()
        full[row0[recv_blk]:row0[recv_blk] + rows[recv_blk]] = rbuf.numpy()


def _ksplit(L, F, row0, rows, me, G):
    acc = None
    for q in range(G):
        j = (me - q) % G
        part = L[:, row0[j]:row0[j] + rows[j]] @ F[row0[j]:row0[j] + rows[j]]
        acc = part if acc is None else acc + part
    return acc


def _worker(rank, world, port, n, p, iters, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2212_02406_b200 as nnb

    parts = [nnb.partition_rows(n, world, g) for g in range(world)]
    row0 = [r0 for r0, _ in parts]
    rows = [r for _, r in parts]
    a = W.gram_shifted(n, seed=5, shift=1.0)
    x0 = W.x0_transpose_norm(a)
    ag = a[row0[rank]:row0[rank] + rows[rank]]
    X = np.zeros((n, n))
    X[row0[rank]:row0[rank] + rows[rank]] = x0[row0[rank]:row0[rank] + rows[rank]]
    R = np.zeros((n, n))
    eps_hist = []
    for k in range(iters + 1):
        _ring_allgather(X, row0, rows, rank, world)
        rg = np.eye(n)[row0[rank]:row0[rank] + rows[rank]] - _ksplit(ag, X, row0, rows, rank, world)
        pair = torch.tensor([np.sum(rg * rg), 0.0], dtype=torch.float64)
        gathered = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, pair)
        ss = 0.0
        for g in range(world):  # rank order
            ss += gathered[g][0].item()
        eps_hist.append(np.sqrt(ss) / np.sqrt(n))
        if k == iters:
            break
        R[row0[rank]:row0[rank] + rows[rank]] = rg
        _ring_allgather(R, row0, rows, rank, world)
        xg = X[row0[rank]:row0[rank] + rows[rank]].copy()
        v = xg
        for _ in range(p):
            v = xg + _ksplit(v, R, row0, rows, rank, world)
        X = np.zeros((n, n))
        X[row0[rank]:row0[rank] + rows[rank]] = v
    out_q.put((rank, row0[rank], X[row0[rank]:row0[rank] + rows[rank]], eps_hist))
    dist.barrier()
    dist.destroy_process_group()


def test_partition_rows_properties():
    import paper_2212_02406_b200 as nnb

    for n in (1, 7, 8, 9, 1000, 32768, 32771):
        for world in (1, 2, 3, 8):
            blocks = [nnb.partition_rows(n, world, g) for g in range(world)]
            assert blocks[0][0] == 0
            for (r0, rs), (r1, _) in zip(blocks, blocks[1:]):
                assert r0 + rs == r1 and (rs == 0 or r0 % 16 == 0)
            assert blocks[-1][0] + blocks[-1][1] == n
            sizes = [rs for _, rs in blocks]
            assert max(sizes) - min(sizes) < 32  # balanced to within two 16-row units


@pytest.mark.parametrize("world", [2])
def test_sharded_schedule_gloo_world2(port, world):
    n, p, iters = 100, 2, 6  # n not a multiple of 8*world: ragged last block
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    portn = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, portn, n, p, iters, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    results.sort()
    X = np.vstack([r[2] for r in results])
    eps = [r[3] for r in results]
    assert all(e == eps[0] for e in eps)  # bit-identical on every rank
    a = W.gram_shifted(n, seed=5, shift=1.0)
    xr, hr, _ = port.chain(a, W.x0_transpose_norm(a), p, iters)
    assert np.linalg.norm(X - xr.real) / np.linalg.norm(xr.real) < 1e-12
    assert np.allclose(eps[0], hr, rtol=1e-9, atol=1e-15)


# ---------------------------------------------------------------- sparse row slabs over gloo
def _sparse_worker(rank, world, port, grid, gamma, theta, out_q):
    """The halo schedule of csrc/sparse_sharded.cu with gloo send/recv and scalar IEEE arithmetic in
    the reference's order (sum += v*x from 0; t = z - theta*y; Z + t; Z*theta)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2212_02406_b200 as nnb

    n = grid * grid
    rp, col, val = W.laplacian_5pt(grid)
    b = W.rhs(n, seed=9)
    r0, rows = nnb.partition_rows(n, world, rank)
    lo, hi = rp[r0], rp[r0 + rows]
    mycols = col[lo:hi]
    h_lo = max(0, r0 - int(mycols.min()))
    h_hi = max(0, int(mycols.max()) - (r0 + rows - 1))
    sizes = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([h_lo, h_hi], dtype=torch.int64))
    send_prev = int(sizes[rank - 1][1]) if rank > 0 else 0
    send_next = int(sizes[rank + 1][0]) if rank < world - 1 else 0

    def exchange(ext):  # ext = [h_lo | own | h_hi]
        reqs, bufs = [], []
        if rank > 0:
            reqs.append(dist.isend(torch.tensor(ext[h_lo:h_lo + send_prev], dtype=torch.float64), rank - 1))
            buf = torch.empty(h_lo, dtype=torch.float64)
            reqs.append(dist.irecv(buf, rank - 1))
            bufs.append((0, buf))
        if rank < world - 1:
            reqs.append(dist.isend(torch.tensor(ext[h_lo + rows - send_next:h_lo + rows], dtype=torch.float64), rank + 1))
            buf = torch.empty(h_hi, dtype=torch.float64)
            reqs.append(dist.irecv(buf, rank + 1))
            bufs.append((h_lo + rows, buf))
        for r in reqs:
            r.wait()
        for off, buf in bufs:
            ext[off:off + len(buf)] = buf.tolist()

    def apply(ext):
        exchange(ext)
        out = [0.0] * rows
        for i in range(rows):
            y = 0.0
            for e in range(rp[r0 + i], rp[r0 + i + 1]):
                y = y + float(val[e]) * ext[int(col[e]) - r0 + h_lo]
            out[i] = ext[h_lo + i] - theta * y
        return out

    pad = lambda own: [0.0] * h_lo + list(own) + [0.0] * h_hi
    z = [float(v) for v in b[r0:r0 + rows]]
    s = 0
    while (1 << s) - 1 < gamma:
        s += 1
    reps = 1
    for _ in range(s):
        t = z
        for _ in range(reps):
            t = apply(pad(t))
        z = [zi + ti for zi, ti in zip(z, t)]
        reps <<= 1
    x = [zi * theta for zi in z]
    out_q.put((rank, r0, x))
    dist.barrier()
    dist.destroy_process_group()


def test_sparse_halo_schedule_gloo_world2(port):
    world, grid, gamma, theta = 2, 12, 15, 0.2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    portn = _free_port()
    procs = [ctx.Process(target=_sparse_worker, args=(r, world, portn, grid, gamma, theta, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    x = np.concatenate([np.array(r[2]) for r in res])
    rp, col, val = W.laplacian_5pt(grid)
    xr, _ = port.sparse_factorized(rp, col, val, W.rhs(grid * grid, seed=9), gamma, theta)
    assert np.array_equal(x, xr.real)  # bit-identical across the partition
