"""Sensor-sharded runs: one process per GPU, NCCL over NVLink.

Counterpart of the reference's ``run_distributed`` (runtime.hpp:768-775),
whose in-process / loopback-TCP message passing gathers every sensor's
contribution at a fusion node and broadcasts the global state back
(runtime.hpp:362-766).  Here the Q sensors are split into contiguous blocks
(rank r owns [r*Q/G, (r+1)*Q/G)), each rank runs the local updates of its
own sensors, one NCCL all-gather per iteration gives every rank every
sensor image, and the fusion step runs redundantly on every rank -- so the
global state, trigger and stopping decision are bitwise identical on all
ranks and no broadcast is needed.  ``torch.distributed`` is only the
rendezvous that ships the 128-byte NCCL unique id.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .api import Hyperparams, Mode, Problem, Solver


def shard_range(q_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous sensor block of ``rank`` (same formula as the C runtime)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    if q_total < 1:
        raise ValueError("Problem: at least one sensor")
    # Q < G: ranks past the sensors get an empty block (they join the
    # exchange and the redundant fusion; C1 beyond 4 GPUs)
    return rank * q_total // world, (rank + 1) * q_total // world


def env_rank_world() -> tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _lib.check(_lib.lib().radmm_nccl_unique_id(buf))
    return bytes(buf)


def broadcast_unique_id(rank: int, world: int) -> bytes | None:
    """Rank 0 creates the NCCL id; torch.distributed ships it to everyone."""
    if world <= 1:
        return None
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def sharded_solver(n_pixels: int, q_total: int, rank: int, world: int, device: int,
                   uid: bytes | None, tcp_timeout_ms: int | None = None) -> Solver:
    b, e = shard_range(q_total, rank, world)
    h = C.c_void_p()
    ids = (C.c_uint8 * 128)(*(uid or bytes(128)))
    _lib.check(_lib.lib().radmm_ctx_create_sharded(device, n_pixels, q_total, b, e, rank, world, ids,
                                                   C.byref(h)))
    if tcp_timeout_ms is not None:
        _lib.check(_lib.lib().radmm_set_transport_timeout(h, int(tcp_timeout_ms)))
    return Solver(n_pixels, e - b, device, _ctx=h, q_total=q_total, q_begin=b)


def run_distributed(problem: Problem, hyper: Hyperparams, mode: Mode = Mode.ASADMM, *,
                    fixed_iterations: bool = False, tcp_timeout_ms: int = 60000):
    """run_distributed (runtime.hpp:768-775) over the torch.distributed world.

    Every rank passes the whole Problem (as the reference does) and uploads
    only its own sensors; every rank returns the same global state (x_G, s,
    sigma, report); ``sensor_images`` holds the rank's own sensors.
    ``tcp_timeout_ms`` keeps the reference's name: a collective or iteration
    that does not complete in time raises TransportError (a dead peer does
    not hang the job).
    """
    problem.validate()
    hyper.validate()
    rank, world, local = env_rank_world()
    uid = broadcast_unique_id(rank, world)
    solver = sharded_solver(problem.pixel_count(), problem.sensor_count(), rank, world, local, uid, tcp_timeout_ms)
    try:
        b, e = shard_range(problem.sensor_count(), rank, world)
        for q in range(b, e):
            solver.set_operator(q - b, problem.operators[q].matrix())
            solver.set_measurement(q - b, problem.measurements[q])
        return solver.run(hyper, mode, fixed_iterations=fixed_iterations)
    finally:
        solver.close()


def fixed_order_mean(images: list) -> np.ndarray:
    """s = (sum_q x_q)/Q in sensor order (admm.hpp:238-240) -- the combine the
    fusion kernel performs on the gathered images on every rank."""
    s = np.zeros_like(images[0])
    for x in images:
        s = s + x
    return (s.view(np.float64) / float(len(images))).view(np.complex128)
