"""Golden vectors for the Sim(3) pose-graph optimisation, produced by the REAL
reference (``patchslam.posegraph`` / ``patchslam.geometry``).  Build container
only (the reference tree does not exist on the GPU box)::

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_pgo.py

Writes ``tests/golden/pgo.npz``:

* ``exp_v`` (20, 7) random tangents -> ``exp_s`` (20, 8) = sim3_exp (geometry.py:303-309),
  ``log_s`` = ``exp_s`` -> ``log_v`` = sim3_log (geometry.py:312-321);
* ``rj_m / rj_a / rj_b`` (30, 8) random similarities -> ``rj_r`` (30, 7),
  ``rj_J`` (30, 7, 7) = residual_and_jacobian (posegraph.py:108-116);
* four ``optimize`` problems (posegraph.py:121-196) built as the reference's
  own tests build them (test_posegraph.py:23-37, 105-179): ``<case>_nodes``,
  ``_odo``, ``_loops`` (k, 2) + ``_loopsim`` (k, 8), ``_maxit``, and the
  results ``_out`` (n, 8), ``_iters``, ``_obj0``, ``_obj``, ``_maxr``,
  ``_conv``, ``_damp``.

Similarities are packed [tx ty tz qx qy qz qw s].
"""

from __future__ import annotations

import os

import numpy as np
from patchslam.geometry import Pose, Similarity, sim3_exp, sim3_log
from patchslam.posegraph import PoseGraphProblem, optimize, residual_and_jacobian

HERE = os.path.dirname(os.path.abspath(__file__))


def pack(sims):
    return np.array([list(s.t) + list(s.q) + [s.s] for s in sims], dtype=np.float64).reshape(-1, 8)


def make_chain(rng, n, step_scale=1.0, translation=0.25, rotation=0.15):
    deltas = []
    nodes = [Similarity.identity()]
    for _ in range(n - 1):
        tangent = np.concatenate([rng.normal(0, translation, 3), rng.normal(0, rotation, 3),
                                  [np.log(step_scale)]])
        delta = sim3_exp(tangent)
        deltas.append(delta)
        nodes.append(nodes[-1] * delta)
    return nodes, deltas


def cases():
    out = {}
    rng = np.random.default_rng(4)
    nodes, deltas = make_chain(rng, 25)
    out["chain"] = ([nodes[0]] + [sim3_exp(rng.normal(0, 0.05, 7)) * s for s in nodes[1:]],
                    deltas, [], 60)
    rng = np.random.default_rng(5)
    nodes, deltas = make_chain(rng, 15)
    loop = (0, 14, nodes[14].inverse() * nodes[0])
    out["loop"] = ([nodes[0]] + [sim3_exp(rng.normal(0, 0.03, 7)) * s for s in nodes[1:]],
                   deltas, [loop], 60)
    rng = np.random.default_rng(7)
    n = 100
    nodes, deltas = make_chain(rng, n, step_scale=1.01)
    loop = (0, n - 1, nodes[n - 1].inverse() * nodes[0])
    out["drift"] = ([Similarity.from_pose(Pose(s.q, s.t)) for s in nodes], deltas, [loop], 100)
    rng = np.random.default_rng(8)
    nodes, deltas = make_chain(rng, 12)
    loops = [(2, 10, sim3_exp(rng.normal(0, 0.2, 7))), (9, 3, sim3_exp(rng.normal(0, 0.2, 7)))]
    out["noisy"] = ([sim3_exp(rng.normal(0, 0.05, 7)) * s for s in nodes], deltas, loops, 30)
    return out


def main():
    z = {}
    rng = np.random.default_rng(123)
    v = rng.normal(0, 0.6, (20, 7))
    v[0] = 0.0
    v[1, 3:6] = 1e-10                    # below the small-angle threshold
    v[2, 3:6] = [np.pi - 1e-3, 0, 0]     # near pi
    sims = [sim3_exp(x) for x in v]
    z["exp_v"] = v
    z["exp_s"] = pack(sims)
    z["log_s"] = pack(sims)
    z["log_v"] = np.array([sim3_log(s) for s in sims])
    ms = [sim3_exp(rng.normal(0, 0.5, 7)) for _ in range(30)]
    sa = [sim3_exp(rng.normal(0, 0.5, 7)) for _ in range(30)]
    sb = [sim3_exp(rng.normal(0, 0.5, 7)) for _ in range(30)]
    rs, js = zip(*[residual_and_jacobian(m, a, b) for m, a, b in zip(ms, sa, sb)])
    z["rj_m"], z["rj_a"], z["rj_b"] = pack(ms), pack(sa), pack(sb)
    z["rj_r"] = np.array(rs)
    z["rj_J"] = np.array(js)
    for name, (nodes, odo, loops, maxit) in cases().items():
        z[f"{name}_nodes"] = pack(nodes)
        z[f"{name}_odo"] = pack(odo)
        z[f"{name}_loops"] = np.array([(j, k) for j, k, _ in loops], dtype=np.int64).reshape(-1, 2)
        z[f"{name}_loopsim"] = pack([d for _, _, d in loops])
        z[f"{name}_maxit"] = np.int64(maxit)
        prob = PoseGraphProblem(list(nodes), list(odo), list(loops))
        rep = optimize(prob, max_iterations=maxit)
        z[f"{name}_out"] = pack(prob.nodes)
        z[f"{name}_iters"] = np.int64(rep.iterations)
        z[f"{name}_obj0"] = np.float64(rep.initial_objective)
        z[f"{name}_obj"] = np.float64(rep.final_objective)
        z[f"{name}_maxr"] = np.float64(rep.max_residual_norm)
        z[f"{name}_conv"] = np.int64(rep.converged)
        z[f"{name}_damp"] = np.float64(prob.damping)
        print(name, rep.iterations, rep.initial_objective, rep.final_objective, rep.converged)
    np.savez_compressed(os.path.join(HERE, "pgo.npz"), **z)


if __name__ == "__main__":
    main()
