"""The N>1 path on CPU: world_size-2 gloo processes.

The CUDA runtime shards sensors across ranks (contiguous blocks), all-gathers
every sensor image once per iteration and runs the fusion redundantly on
every rank (radmm_b200.cu: exchange/build_contrib/run_fusion).  These tests
drive the same decomposition with the CPU oracle as the per-rank compute and
torch.distributed (gloo) as the exchange, and require the sharded run to be
bitwise identical to the single-process run -- the property the fixed-order
sum over the gathered images guarantees at any rank count.  They also cover
the host plumbing the GPU path uses: the NCCL unique-id broadcast and the
lambda max-reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_08606_b200.distributed import fixed_order_mean, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(Q=5):
    from paper_2307_08606_b200 import scenario
    cfg = scenario.baseline_config("c1", nside=12, K=16, n_targets=5, max_iter=80, Q=Q)
    ops, ys, _, hyper = scenario.baseline_problem(cfg)
    hyper["screening_tol"] = 1e-3  # make elimination fire inside 80 iterations
    return [a.astype(np.complex128) for a in ops], ys, hyper


def _sharded_oracle_run(rank, world, port, out, Q_total=5):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle import admm_ref as R
    ops, ys, hyper = _problem(Q_total)
    h = R.Hyper(**hyper)
    Q, N = len(ops), ops[0].shape[1]
    b, e = shard_range(Q, rank, world)
    sensors = [R.SensorRef(ops[q], ys[q], h) for q in range(b, e)]
    qmax = -(-Q // world)
    fusion = R.FusionRef(N, Q, h)
    staged = False
    xs, sizes = [], []
    for k in range(1, h.max_iter + 1):
        if staged:
            for s in sensors:
                s.screen()
        for s in sensors:
            s.local_update(fusion.gap, fusion.sigma)
        send = torch.zeros((qmax, 2 * N), dtype=torch.float64)
        for i, s in enumerate(sensors):
            send[i] = torch.from_numpy(s.x_full.view(np.float64).copy())
        recv = [torch.zeros_like(send) for _ in range(world)]
        dist.all_gather(recv, send)
        images = []
        for r in range(world):
            rb, re_ = shard_range(Q, r, world)
            for i in range(re_ - rb):
                images.append(recv[r][i].numpy().copy().view(np.complex128))
        for q, img in enumerate(images):
            fusion.contrib[q] = img
        fusion.round()
        # the fusion kernel's combine is the fixed-order mean of the gathered images
        assert np.array_equal(fusion.s, fixed_order_mean(images))
        sizes.append([s.active.size for s in sensors])
        staged = fusion.trigger
    # records: each rank logs its own sensors' sizes per iteration and ONE
    # all-gather at the end of the run assembles the global table
    # (finish_sharded_records in the CUDA runtime)
    meta = torch.zeros((len(sizes), qmax), dtype=torch.float64)
    for k, row in enumerate(sizes):
        for i, v in enumerate(row):
            meta[k, i] = v
    gathered = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(gathered, meta)
    table = [[int(gathered[r][k, i]) for r in range(world)
              for i in range(shard_range(Q, r, world)[1] - shard_range(Q, r, world)[0])] for k in range(len(sizes))]
    lam = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(lam, op=dist.ReduceOp.MAX)
    obj = [b"uid-from-rank0" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    out[rank] = {"x_global": fusion.x_g, "s": fusion.s, "sigma": fusion.sigma, "sizes": sizes,
                 "lam": float(lam.item()), "uid": obj[0], "x_local": [s.x_full for s in sensors], "table": table}
    dist.destroy_process_group()


def test_shard_range_partition():
    """Contiguous blocks covering every sensor once; Q < G leaves the ranks
    past the sensors with empty blocks (config 1 on 8 GPUs)."""
    with pytest.raises(ValueError):
        shard_range(0, 0, 2)
    for Q in (1, 4, 5, 8, 32):
        for G in (1, 2, 3, 4, 8):
            blocks = [shard_range(Q, r, G) for r in range(G)]
            assert blocks[0][0] == 0 and blocks[-1][1] == Q
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            assert max(e - b for b, e in blocks) - min(e - b for b, e in blocks) <= 1


def test_two_rank_gloo_run_is_bitwise_identical_to_single_process():
    from oracle import admm_ref as R
    ops, ys, hyper = _problem()
    ref = R.run(ops, ys, R.Hyper(**hyper), asadmm=True, fixed_iterations=True)
    assert any(rec.active_sizes != ref.records[0].active_sizes for rec in ref.records)  # elimination fired
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sharded_oracle_run, args=(2, port, out), nprocs=2, join=True)
    for rank in range(2):
        o = out[rank]
        assert np.array_equal(o["x_global"], ref.x_global)
        assert np.array_equal(o["s"], ref.s)
        assert np.array_equal(o["sigma"], ref.sigma)
        assert o["lam"] == 2.0 and o["uid"] == b"uid-from-rank0"
        b, e = shard_range(len(ops), rank, 2)
        for i, q in enumerate(range(b, e)):
            assert np.array_equal(o["x_local"][i], ref.sensor_images[q])
            assert [sz[i] for sz in o["sizes"]] == [rec.active_sizes[q] for rec in ref.records]


def test_end_of_run_records_and_idle_ranks():
    """Q = 2 sensors on 3 ranks (one rank holds none): the run is
    bitwise the single-process one, and the per-iteration active-size table
    assembled by one all-gather at the end of the run equals its records."""
    from oracle import admm_ref as R
    ops, ys, hyper = _problem(2)
    ref = R.run(ops, ys, R.Hyper(**hyper), asadmm=True, fixed_iterations=True)
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sharded_oracle_run, args=(3, port, out, 2), nprocs=3, join=True)
    for rank in range(3):
        o = out[rank]
        assert np.array_equal(o["s"], ref.s) and np.array_equal(o["sigma"], ref.sigma)
        assert o["table"] == [list(rec.active_sizes) for rec in ref.records]
    assert sorted(len(out[r]["x_local"]) for r in range(3)) == [0, 1, 1]
