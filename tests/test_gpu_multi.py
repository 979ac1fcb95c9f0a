"""Multi-GPU sharded CUDA run (NCCL over NVLink) against the single-GPU run
and the oracle.  Needs >= 2 visible GPUs (skipped otherwise: the gpurun pool
gives one); the decomposition itself is covered on CPU by
tests/test_distributed_cpu.py and the one-rank NCCL path by
test_gpu_parity.py::test_nccl_exchange_path_one_rank_equals_plain.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from paper_2307_08606_b200 import scenario
    cfg = scenario.baseline_config("c1", nside=24, K=32, n_targets=6, max_iter=60, Q=5)
    ops, ys, _, hyper = scenario.baseline_problem(cfg)
    hyper["screening_tol"] = 1e-3
    return ops, ys, hyper


def _rank(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2307_08606_b200 import api, distributed as D
    ops, ys, hyper = _problem()
    prob = api.Problem([api.ForwardOperator.from_matrix(a) for a in ops], ys)
    r = D.run_distributed(prob, api.Hyperparams(**hyper), api.Mode.ASADMM, fixed_iterations=True)
    out[rank] = {"s": r.s, "sigma": r.sigma, "x_global": r.x_global, "iters": r.iterations,
                 "sizes": [list(it.active_sizes) for it in r.report.iterations],
                 "bytes": [it.bytes_sent for it in r.report.iterations], "images": r.sensor_images}
    dist.destroy_process_group()


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_run_equals_single_gpu(world, built_lib):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    from paper_2307_08606_b200 import api
    ops, ys, hyper = _problem()
    single = api.run(api.Problem([api.ForwardOperator.from_matrix(a) for a in ops], ys), api.Hyperparams(**hyper),
                     api.Mode.ASADMM, fixed_iterations=True)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        o = out[r]
        # fixed-order sum over the gathered images: bitwise equal at any rank count
        assert np.array_equal(o["s"], single.s) and np.array_equal(o["sigma"], single.sigma)
        assert o["sizes"] == [list(it.active_sizes) for it in single.report.iterations]
        assert o["bytes"] == [it.bytes_sent for it in single.report.iterations]
