"""The row-strip decomposition of DESIGN.md section 9 on CPU (gloo, world_size 2/3).

Each rank owns the rows `csph_strip_rows` gives it (the product's partition
function, host code), keeps 3 ghost rows per side, and per step: allreduce-max of
the Eq.7 maxima -> tau, one step of R on its strip, then swaps its 3
edge rows with ranks r-1, r+1 (no wrap, reading #18).  The strip arithmetic is the
oracle's, so this checks the decomposition design itself: a 3-row halo and a max
allreduce reproduce the single-domain result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEPS = 25


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _strip_rows(ny, n, r):
    from paper_2103_15196_b200 import csph
    return csph.csph_strip_rows(ny, n, r)


def _worker(rank, world, port, cfg, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    name, nx, ny = cfg
    c = synth.config(name, nx, ny)
    h, hu, hv, b, psi = synth.fill(c)
    j0, j1 = _strip_rows(ny, world, rank)
    rows = j1 - j0
    G = oracle.GHOST
    # padded window rows j0-3 .. j1+3 (rows outside the grid are wall ghosts, filled
    # by the oracle's mirror on wall sides)
    def window(a, fill=0.0):
        out = np.full((rows + 2 * G, nx + 2 * G), fill)
        lo, hi = max(0, j0 - G), min(ny, j1 + G)
        out[lo - (j0 - G):hi - (j0 - G), G:G + nx] = a[lo:hi]
        return out
    W = 1.0 / (1.0 - psi)
    o = oracle.Oracle(nx, rows, c.dx, oracle.Params(**c.params))
    o.set_walls(True, True, rank == 0, rank == world - 1)
    o.set_state_padded(window(h), window(hu), window(hv), window(b), window(W, 1.0))
    Wp = o.debug("W")
    dts = []
    for _ in range(STEPS):
        M = torch.tensor(o.reduce_M())
        dist.all_reduce(M, op=dist.ReduceOp.MAX)
        st, tau, lim = o.tau_from_M(M.numpy())
        assert st == 0
        dts.append(tau)
        assert o.step_tau(tau) == 0
        H, Qx, Qy, bb = [np.ascontiguousarray(x) for x in o.get_state_padded()]
        fields = [H, Qx, Qy, bb]
        reqs = []
        recv = {}
        for k, f in enumerate(fields):
            if rank > 0:
                reqs.append(dist.isend(torch.from_numpy(f[G:2 * G].copy()), rank - 1, tag=10 + k))
                recv[(k, "lo")] = torch.empty((G, nx + 2 * G), dtype=torch.float64)
                reqs.append(dist.irecv(recv[(k, "lo")], rank - 1, tag=20 + k))
            if rank < world - 1:
                reqs.append(dist.isend(torch.from_numpy(f[rows:rows + G].copy()), rank + 1, tag=20 + k))
                recv[(k, "hi")] = torch.empty((G, nx + 2 * G), dtype=torch.float64)
                reqs.append(dist.irecv(recv[(k, "hi")], rank + 1, tag=10 + k))
        for r in reqs:
            r.wait()
        for (k, side), t in recv.items():
            if side == "lo":
                fields[k][0:G] = t.numpy()
            else:
                fields[k][rows + G:rows + 2 * G] = t.numpy()
        o.set_state_padded(*fields, Wp)
    own = [np.ascontiguousarray(x) for x in o.get_state()]
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), h=own[0], hu=own[1], hv=own[2], b=own[3],
             dt=np.array(dts), j0=j0, j1=j1)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [(2, ("C4", 40, 37)), (3, ("C3", 36, 44))])
def test_strip_decomposition_bitwise(tmp_path, world, cfg):
    name, nx, ny = cfg
    c = synth.config(name, nx, ny)
    ref = oracle.Oracle(nx, ny, c.dx, oracle.Params(**c.params))
    ref.set_state(*synth.fill(c))
    st, dt_ref, _ = ref.step(STEPS)
    assert st == 0
    H, Qx, Qy, b = ref.get_state()
    mp.spawn(_worker, args=(world, _free_port(), cfg, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        j0, j1 = int(d["j0"]), int(d["j1"])
        assert np.array_equal(d["dt"], dt_ref)
        assert np.array_equal(d["h"], H[j0:j1]) and np.array_equal(d["b"], b[j0:j1])
        assert np.array_equal(d["hu"], Qx[j0:j1]) and np.array_equal(d["hv"], Qy[j0:j1])


def _bounds_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    import bench
    c = synth.config("C5", 600, 700)
    b = bench.strip_bounds(c, c.ny, c.nx, world, rank, "balanced", "cpu")
    np.save(os.path.join(out_dir, f"b{rank}.npy"), np.array(b))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_balanced_partition(tmp_path, world):
    """bench.py's load-balanced strips: every rank derives the same bounds
    from all-gathered wet-row counts, equal to csph_balance_rows on the whole field."""
    from paper_2103_15196_b200 import csph
    c = synth.config("C5", 600, 700)
    h = synth.fill(c)[0]
    w = (h > 1e-6).sum(axis=1).astype(np.float64) + 0.03 * c.nx
    ref = csph.csph_balance_rows(c.ny, world, w)
    mp.spawn(_bounds_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.load(tmp_path / f"b{r}.npy").tolist() == ref
    per = [w[ref[r]:ref[r + 1]].sum() for r in range(world)]
    even = [w[csph.csph_strip_rows(c.ny, world, r)[0]:csph.csph_strip_rows(c.ny, world, r)[1]].sum()
            for r in range(world)]
    assert max(per) <= max(even) + 1e-9
