"""Shared parity helpers: run the CUDA path and the CPU oracle on the same inputs."""
from __future__ import annotations

import numpy as np

from oracle import admm_ref
from paper_2307_08606_b200 import api


def quantize(ops):
    """The device stores operators as complex64; the oracle sees the same values."""
    return [np.asarray(a).astype(np.complex64) for a in ops]


def gpu_run(ops64, ys, hyper: dict, asadmm=True, **kw):
    prob = api.Problem([api.ForwardOperator.from_matrix(a) for a in ops64], ys)
    return api.run(prob, api.Hyperparams(**hyper), api.Mode.ASADMM if asadmm else api.Mode.SADMM, **kw)


def oracle_run(ops64, ys, hyper: dict, asadmm=True, **kw):
    return admm_ref.run([a.astype(np.complex128) for a in ops64], ys, admm_ref.Hyper(**hyper),
                        asadmm=asadmm, **kw)


def rel(a, b) -> float:
    return admm_ref.relative_l2_diff(np.asarray(a).ravel(), np.asarray(b).ravel())


def state_errors(g, o) -> dict:
    return {
        "x_global": rel(g.x_global, o.x_global),
        "s": rel(g.s, o.s),
        "sigma": rel(g.sigma, o.sigma),
        "sensor_images": rel(np.concatenate(g.sensor_images), np.concatenate(o.sensor_images)),
        "image": rel(g.image, o.image),
    }


def gpu_masks(g, q_count):
    """{(iteration, sensor): sorted removed pixels} from the GPU removal log."""
    out = {}
    for k, q, p in g.removal_log:
        out.setdefault((int(k), int(q)), []).append(int(p))
    return {key: np.array(sorted(v)) for key, v in out.items()}


def oracle_masks(o):
    return {(e.iteration, e.sensor): np.sort(e.removed) for e in o.events if e.removed.size}


def compare_masks(g, o, tol: float, window: int, rel_bound: float = 1e-9):
    """Mask parity: identical removal sets except pixels whose criterion sits
    within round-off of the threshold; returns (mismatched_pixels, near_threshold)."""
    gm, om = gpu_masks(g, None), oracle_masks(o)
    zeta = {(e.iteration, e.sensor): (e.active_before, e.zeta) for e in o.events}
    bad, near = 0, 0
    for key in set(gm) | set(om):
        a = set(gm.get(key, np.array([], int)).tolist())
        b = set(om.get(key, np.array([], int)).tolist())
        for p in a ^ b:
            act, z = zeta.get(key, (None, None))
            if z is not None and p in set(act.tolist()):
                zj = z[list(act).index(p)]
                if abs(zj - tol) <= rel_bound * max(tol, abs(zj)):
                    near += 1
                    continue
            bad += 1
    return bad, near
