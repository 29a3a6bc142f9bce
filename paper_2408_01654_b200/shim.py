"""Install this package as the hot path of an existing ``patchslam`` process.

    from paper_2408_01654_b200 import shim
    restore = shim.install()          # patchslam now runs BA / reprojection on the B200
    ...
    restore()                         # put the reference functions back

The reference dispatches by module attribute, and several modules import the
hot-path functions BY NAME, so replacing the canonical definitions is not
enough (verified with a call-counting probe):

* ``reproject_grid`` is bound by name in ``patchslam.ba`` (ba.py:24-33),
  ``patchslam.graph`` (graph.py:29-38) and ``patchslam.synthetic``
  (synthetic.py:17-25) besides ``patchslam.geometry``;
* ``block_cholesky`` is bound by name in ``patchslam.ba`` (ba.py:22);
* ``ba._BACKENDS`` (ba.py:490) holds the original solver objects;
* the pose-graph functions (``patchslam.posegraph``) are replaced by the
  device versions of ``posegraph.py`` here.

``loop``, ``pipeline`` and ``cli`` use ``from . import ba`` plus attribute
access, so they follow the patched module.  Exceptions need no mapping: when
``patchslam`` is importable this package's error classes derive from the
reference's (errors.py), so the reference's ``except SingularSystem`` catches
them.  Modules imported with ``from patchslam.x import f`` AFTER install()
get this package's function; ones imported before keep the reference's.
"""

from __future__ import annotations

import importlib

BA_NAMES = ("BAProblem", "residuals", "objective", "assemble", "solve", "solve_dense",
            "solve_block_sparse", "_apply_step", "select_backend")
# Sim(3) pose-graph optimisation (posegraph.py:85-196); PoseGraphProblem and
# the reference value types stay: the device functions accept them
PGO_NAMES = ("objective", "residual_smooth", "residual_loop", "residual_and_jacobian", "optimize")


def install():
    """Patch the reference modules in place; returns a zero-argument restore()."""
    from . import ba, block_cholesky, geometry, posegraph
    rba = importlib.import_module("patchslam.ba")
    rpg = importlib.import_module("patchslam.posegraph")
    rgeo = importlib.import_module("patchslam.geometry")
    rgraph = importlib.import_module("patchslam.graph")
    rsyn = importlib.import_module("patchslam.synthetic")
    rbc = importlib.import_module("patchslam.block_cholesky")
    saved = []

    def put(mod, name, value):
        saved.append((mod, name, getattr(mod, name)))
        setattr(mod, name, value)

    for mod in (rgeo, rgraph, rsyn, rba):
        put(mod, "reproject_grid", geometry.reproject_grid)
    for name in BA_NAMES:
        put(rba, name, getattr(ba, name))
    for name in PGO_NAMES:
        put(rpg, name, getattr(posegraph, name))
    put(rba, "block_cholesky", block_cholesky.block_cholesky)
    put(rbc, "block_cholesky", block_cholesky.block_cholesky)
    backends = dict(rba._BACKENDS)
    rba._BACKENDS[rba.DENSE] = ba.solve_dense
    rba._BACKENDS[rba.BLOCK_SPARSE] = ba.solve_block_sparse

    def restore():
        for mod, name, value in reversed(saved):
            setattr(mod, name, value)
        rba._BACKENDS.clear()
        rba._BACKENDS.update(backends)
    return restore
