"""World-size-2 gloo tests of the multi-process path on CPU.

Covered here without a GPU: the NCCL-id bootstrap over torch.distributed, the shard rule
on every rank (from libtfdp), max-over-ranks timing, and the data flow of one exact-path
iteration — each rank evaluates its own targets against all sources (the oracle stands in
for the kernels, which need a GPU), updates its slice, and the slices are all-gathered —
reproducing the single-process iteration bit for bit (R15)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import oracle as O
    import paper_2303_03964_b200 as P
    from paper_2303_03964_b200 import dist as D
    from synth import make_config

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # 1) NCCL-id bootstrap: rank 0's id reaches every rank unchanged
        fake = bytes((7 * i + 3) % 256 for i in range(128))
        d = D.bootstrap(device=0, uid_fn=lambda: fake)
        out["uid_ok"] = d is not None and bytes(d._uid) == fake and (d.rank, d.world) == (rank, world)
        # 2) shard rule from the library
        w = make_config("C2rgg")
        lo, hi = D.my_shard(w.n)
        out["shard"] = (lo, hi)
        # 3) max over ranks
        out["max"] = D.max_over_ranks(float(rank + 1))
        # 4) one sharded exact iteration + all-gather of the updated slices
        rp, col = O.csr_build(w.n, w.u, w.v)
        X = w.xy.astype(np.float64)
        idx = np.arange(lo, hi)
        R, A = O.forces_exact(X, rp, col, O.Params(), targets=idx)
        mine = torch.from_numpy(X[lo:hi] + O.eta(0, 300) * (R + A))
        sizes = [P.shard_range(w.n, world, r) for r in range(world)]
        bufs = [torch.zeros((b - a, 2), dtype=torch.float64) for a, b in sizes]
        for r in range(world):  # the library's exchange: one broadcast per shard (unequal sizes)
            if r == rank:
                bufs[r].copy_(mine)
            dist.broadcast(bufs[r], src=r)
        Xn = torch.cat(bufs).numpy()
        ref = O.step(X, rp, col, O.Params(), O.eta(0, 300))
        out["step_bitwise"] = bool(np.array_equal(Xn, ref))
        # 5) slab mode of the ibFFT path: the library's plan is identical on
        # every rank, partitions rows and half-spectrum columns, and the two transposes it
        # implies (row slabs -> column chunks -> row slabs), carried over gloo here, deliver
        # to every rank exactly its block of the half spectra
        rows, Pf = 1003 * 3, 6144
        row0, q0 = P.slab_plan(rows, Pf, world)
        out["plan"] = (row0, q0)
        R_, H = row0[-1], Pf // 2 + 1
        full = np.random.default_rng(5).standard_normal((3, R_, H)).astype(np.float32)
        mine_rows = slice(row0[rank], row0[rank + 1])
        segs = {s: full[:, mine_rows, q0[s]:q0[s + 1]].copy() for s in range(world)}
        got = [None] * world
        dist.all_gather_object(got, segs)  # message (r -> s) = got[r][s]
        xb = np.concatenate([got[r][rank] for r in range(world)], axis=1)
        out["cols_ok"] = bool(np.array_equal(xb, full[:, :, q0[rank]:q0[rank + 1]]))
        back = {r: 2.0 * xb[:, row0[r]:row0[r + 1], :] for r in range(world)}  # "column pass"
        got = [None] * world
        dist.all_gather_object(got, back)
        rows_back = np.concatenate([got[s][rank] for s in range(world)], axis=2)
        out["rows_ok"] = bool(np.array_equal(rows_back, 2.0 * full[:, mine_rows, :]))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_multiprocess_path(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle as O
    from synth import make_config

    n = make_config("C2rgg").n
    for r in range(world):
        assert res[r]["uid_ok"]
        assert res[r]["shard"] == O.shard_range(n, world, r)
        assert res[r]["max"] == float(world)
        assert res[r]["step_bitwise"]
        assert res[r]["cols_ok"] and res[r]["rows_ok"]
        assert res[r]["plan"] == res[0]["plan"]
