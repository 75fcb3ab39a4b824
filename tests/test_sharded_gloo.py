"""World-size-2 CPU (gloo) coverage of the row-sharded schedule.

The NCCL path itself needs GPUs; here two processes run the SAME schedule as
paper_2212_02406_b200/csrc/sharded.cu with torch.distributed (gloo) standing in
for NCCL and numpy for the local DMMA GEMMs:
  * row blocks from the library's own nnb_partition_rows (16-row units),
  * ring all-gather in G-1 send/recv steps, partial products own block first
    then in ring order (K split by the ranks' row blocks),
  * eps from the per-rank Σ‖R_g‖² all-gathered and summed in rank order.
Checked against the single-process oracle chain and for bit-identical eps on
every rank (identical stop decisions).  The int8-emulated products of the same
file (column statistics gathered and combined in rank order, residue blocks on
the ring, K-block products accumulated mod m) are restated with integer numpy
and checked against the whole product's residues; the sparse halo schedules (a
halo per application, and the temporal-blocked slabs with one halo exchange per pass)
are checked bit-exact against the reference."""
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


# ---------------------------------------------------------------- int8-emulated products over gloo
_MODULI = (256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199)


def _exp_for(amax):
    """2^e·amax in [2^52, 2^53) (ozaki.cu exp_for)."""
    return 0 if amax == 0.0 else 52 - (np.frexp(amax)[1] - 1)


def _residues(ints, s):
    """Signed residues in [-128, 127] of exact integers (int64 array) for the first s moduli."""
    out = []
    for m in _MODULI[:s]:
        r = np.mod(ints, m)
        r = np.where(r > 127, r - m, r)
        out.append(r.astype(np.int64))
    return out


def _oz_worker(rank, world, port, n, s, out_q):
    """csrc/sharded.cu's int8-emulated product C_g = L_g·F with F row-sharded, restated with
    gloo for NCCL and numpy integers for the int8 GEMMs:
      * per-column [max|x|, Σ|x|, Σx²] of the rank's rows, all-gathered, combined in rank order;
      * the rank's block of F scaled by the global column exponents and split into residues;
      * a ring all-gather of the residue blocks (same step order as oz_ring);
      * G K-block products accumulated mod m, own block first then ring order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2212_02406_b200 as nnb

    parts = [nnb.partition_rows(n, world, g) for g in range(world)]
    row0 = [r0 for r0, _ in parts]
    rows = [r for _, r in parts]
    rng = np.random.default_rng(11)
    L = rng.standard_normal((n, n)) * np.exp(rng.uniform(-3, 3, (n, 1)))
    F = rng.standard_normal((n, n)) * np.exp(rng.uniform(-3, 3, (1, n)))
    me = rank
    fg = F[row0[me]:row0[me] + rows[me]]
    # 1. column statistics of the own rows, gathered and combined in rank order
    rec = torch.from_numpy(np.concatenate([np.abs(fg).max(axis=0, initial=0.0), np.abs(fg).sum(axis=0),
                                           (fg * fg).sum(axis=0)]))
    recs = [torch.zeros(3 * n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(recs, rec)
    colmax = np.zeros(n)
    for g in range(world):
        colmax = np.maximum(colmax, recs[g][:n].numpy())
    eb = np.array([_exp_for(v) for v in colmax])
    # 2. own block scaled and split
    fb = np.rint(np.ldexp(fg, eb[None, :])).astype(np.int64)
    blocks = {me: _residues(fb, s)}
    # 3. ring of residue blocks
    for q in range(1, world):
        send_blk, recv_blk = (me - q + 1) % world, (me - q) % world
        sbuf = torch.from_numpy(np.stack(blocks[send_blk]).astype(np.int8))
        rbuf = torch.empty((s, rows[recv_blk], n), dtype=torch.int8)
        reqs = [dist.isend(sbuf, (me + 1) % world), dist.irecv(rbuf, (me - 1) % world)]
        for r in reqs:
            r.wait()
        blocks[recv_blk] = [rbuf[l].numpy().astype(np.int64) for l in range(s)]
    # 4. the rank's rows of L, its row exponents and residues; K-block products mod m
    lg = L[row0[me]:row0[me] + rows[me]]
    ea = np.array([_exp_for(v) for v in np.abs(lg).max(axis=1, initial=0.0)])
    la = _residues(np.rint(np.ldexp(lg, ea[:, None])).astype(np.int64), s)
    acc = [None] * s
    for q in range(world):
        j = (me - q) % world
        for l, m in enumerate(_MODULI[:s]):
            part = np.mod(la[l][:, row0[j]:row0[j] + rows[j]] @ blocks[j][l], m)
            acc[l] = part if acc[l] is None else np.mod(acc[l] + part, m)
    out_q.put((rank, row0[me], eb, ea, np.stack(acc)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_int8_emulated_product_schedule_gloo(world):
    """The sharded residue schedule reproduces the whole product's residues exactly: the
    global column exponents and, per modulus, (A'·B') mod m of the unsharded scaled operands."""
    n, s = 72, 4  # 72 rows: 16-row units give ragged blocks (48/24 at world 2, 32/32/8 at world 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    portn = _free_port()
    procs = [ctx.Process(target=_oz_worker, args=(r, world, portn, n, s, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    rng = np.random.default_rng(11)
    L = rng.standard_normal((n, n)) * np.exp(rng.uniform(-3, 3, (n, 1)))
    F = rng.standard_normal((n, n)) * np.exp(rng.uniform(-3, 3, (1, n)))
    eb = np.array([_exp_for(v) for v in np.abs(F).max(axis=0)])
    ea = np.array([_exp_for(v) for v in np.abs(L).max(axis=1)])
    A = np.rint(np.ldexp(L, ea[:, None])).astype(np.int64)
    B = np.rint(np.ldexp(F, eb[None, :])).astype(np.int64)
    la, fb = _residues(A, s), _residues(B, s)
    for rank, r0, eb_r, ea_r, acc in res:
        assert np.array_equal(eb_r, eb)  # every rank: the global column exponents
        rows = acc.shape[1]
        assert np.array_equal(ea_r, ea[r0:r0 + rows])
        for l, m in enumerate(_MODULI[:s]):
            whole = np.mod(la[l][r0:r0 + rows] @ fb[l], m)
            assert np.array_equal(acc[l], whole)
    # and the residues are those of the exact integer product A'·B' (CRT-consistent)
    prod = A[:8].astype(object) @ B.astype(object)
    for l, m in enumerate(_MODULI[:s]):
        assert np.array_equal(np.mod(prod, m).astype(np.int64), res[0][4][l][:8])


# ---------------------------------------------------------------- temporal-blocked slabs over gloo
def _tb_worker(rank, world, port, grid, gamma, theta, out_q):
    """sparse_sharded.cu's temporal-blocked slab schedule (run_slabs_tb) restated with gloo and
    scalar IEEE arithmetic in the reference's order: per pass of up to D applications (D = 8,
    sparse.cuh kStencilDepthSlab) the D halo grid rows of its input are exchanged once, the pass runs over the slab's extended
    rows (cells past them read as zero, so the halo goes stale one row per application and
    never reaches the own rows), and only the own rows are kept."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2212_02406_b200 as nnb

    W_, n = grid, grid * grid
    rp, col, val = W.laplacian_5pt(grid)
    b = W.rhs(n, seed=13)
    r0, rows = nnb.partition_rows(n, world, rank)
    D = 8  # applications per pass = halo grid rows
    assert r0 % W_ == 0 and rows % W_ == 0 and rows >= D * W_
    hw = D * W_
    lo = hw if rank > 0 else 0
    hi = hw if rank < world - 1 else 0
    e0 = r0 - lo  # global index of the extended region's first cell

    def exchange(ext):
        reqs, bufs = [], []
        if rank > 0:
            reqs.append(dist.isend(torch.tensor(ext[lo:lo + hw], dtype=torch.float64), rank - 1))
            bb = torch.empty(hw, dtype=torch.float64)
            reqs.append(dist.irecv(bb, rank - 1))
            bufs.append((0, bb))
        if rank < world - 1:
            reqs.append(dist.isend(torch.tensor(ext[lo + rows - hw:lo + rows], dtype=torch.float64), rank + 1))
            bb = torch.empty(hw, dtype=torch.float64)
            reqs.append(dist.irecv(bb, rank + 1))
            bufs.append((lo + rows, bb))
        for r in reqs:
            r.wait()
        for off, bb in bufs:
            ext[off:off + hw] = bb.tolist()

    def step(ext):
        out = list(ext)
        for i in range(len(ext)):
            g = e0 + i
            y = 0.0
            for e in range(rp[g], rp[g + 1]):
                j = int(col[e]) - e0
                y = y + float(val[e]) * (ext[j] if 0 <= j < len(ext) else 0.0)
            out[i] = ext[i] - theta * y
        return out

    ext_len = lo + rows + hi
    z = [0.0] * ext_len
    z[lo:lo + rows] = [float(v) for v in b[r0:r0 + rows]]
    s_f = 0
    while (1 << s_f) - 1 < gamma:
        s_f += 1
    for f in range(s_f):
        left, t = 1 << f, list(z)
        while left > 0:
            steps = min(D, left)
            left -= steps
            exchange(t)
            for _ in range(steps):
                t = step(t)
        z = [zi + ti for zi, ti in zip(z, t)]
    x = [zi * theta for zi in z[lo:lo + rows]]
    out_q.put((rank, r0, x))
    dist.barrier()
    dist.destroy_process_group()


def test_sparse_temporal_blocked_slabs_gloo_world2(port):
    world, grid, gamma, theta = 2, 32, 15, 0.2  # 2 slabs of 16 grid rows, 8-row halos
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    portn = _free_port()
    procs = [ctx.Process(target=_tb_worker, args=(r, world, portn, grid, gamma, theta, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    x = np.concatenate([np.array(r[2]) for r in res])
    rp, col, val = W.laplacian_5pt(grid)
    xr, _ = port.sparse_factorized(rp, col, val, W.rhs(grid * grid, seed=13), gamma, theta)
    assert np.array_equal(x, xr.real)  # bit-identical: the halo never reaches the own rows
