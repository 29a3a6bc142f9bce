"""Patch-graph text fixtures: the reference's line format (graph.py:9-20),
written and parsed over the structure-of-arrays graph.

Records, one per line (``#`` comments and blank lines ignored)::

    meta patch_size <p>
    intrinsics <fx> <fy> <cx> <cy>
    frame <id> <timestamp> <keyframe 0|1> <features 0|1> <tx> <ty> <tz> <qx> <qy> <qz> <qw>
    patch <frame> <index> <inverse_depth> <landmark|-1> <x0> <y0> ...   (p*p pairs)
    edge <src_frame> <src_patch> <dst_frame> <odometry|loop> <wx> <wy> <tx0> <ty0> ...

Floats use ``repr`` so a write/read round trip is bit-exact (SURVEY 8(f)
rank 3: fixtures as the golden-input interchange between the CPU reference
and the GPU path).  Behaviour follows graph.py:264-357: unknown record kinds
are returned as ``(line number, tokens)`` extras (scene fixtures append
``landmark`` records), malformed records and a missing intrinsics record
raise ParseError with the file and line, frame ids must be contiguous from
0, patches are ordered by index inside their frame, every edge is checked
against the frames and patches it references, and poses pass through Pose
(quaternion re-normalisation) exactly as the reference's parser does.
"""

from __future__ import annotations

import numpy as np

from .errors import ParseError
from .geometry import DEFAULT_PATCH_SIZE, Intrinsics, Pose
from .graph import _KIND_CODE, _KIND_NAME, LOOP, PatchGraph


def _f(x) -> str:
    return repr(float(x))


def graph_to_lines(graph: PatchGraph) -> list[str]:
    """Fixture lines of a graph (graph.py:268-288 record order: header, meta,
    intrinsics, frames, patches frame-major, edges in graph order)."""
    k = graph.intrinsics
    out = ["# patchgraph v1", f"meta patch_size {graph.patch_size}",
           "intrinsics " + " ".join(_f(v) for v in (k.fx, k.fy, k.cx, k.cy))]
    q, t = graph._q.view, graph._t.view
    ts, kf, feat = graph._ts.view, graph._kf.view, graph._feat.view
    for f in range(graph.n_frames):
        out.append(f"frame {f} {_f(ts[f])} {int(bool(kf[f]))} {int(bool(feat[f]))} "
                   + " ".join(_f(v) for v in np.concatenate([t[f], q[f]])))
    off = graph.patch_offset()
    grid, depth, lm = graph._grid.view, graph._depth.view, graph._lm.view
    for f in range(graph.n_frames):
        for idx in range(int(off[f + 1] - off[f])):
            g = int(off[f]) + idx
            out.append(f"patch {f} {idx} {_f(depth[g])} {int(lm[g])} "
                       + " ".join(_f(v) for v in grid[g].ravel()))
    src, pat, dst = graph._src.view, graph._pat.view, graph._dst.view
    conf, tgt, kind = graph._conf.view, graph._tgt.view, graph._kind.view
    for e in range(graph.n_edges):
        out.append(f"edge {int(src[e])} {int(pat[e])} {int(dst[e])} {_KIND_NAME[int(kind[e])]} "
                   + " ".join(_f(v) for v in conf[e]) + " "
                   + " ".join(_f(v) for v in tgt[e].ravel()))
    return out


def write_graph(graph: PatchGraph, path, extra_lines=()) -> None:
    with open(path, "w") as fh:
        for line in graph_to_lines(graph):
            fh.write(line + "\n")
        for line in extra_lines:
            fh.write(line + "\n")


def parse_graph_lines(lines, path: str | None = None):
    """Parse fixture lines into (PatchGraph, extras)."""
    intr = None
    p = DEFAULT_PATCH_SIZE
    frames, patches, edges, extras = [], [], [], []
    for ln, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        tok = line.split()
        head = tok[0]
        try:
            if head == "meta" and tok[1] == "patch_size":
                p = int(tok[2])
            elif head == "intrinsics":
                intr = Intrinsics(*(float(v) for v in tok[1:5]))
            elif head == "frame":
                frames.append((int(tok[1]), float(tok[2]), bool(int(tok[3])), bool(int(tok[4])),
                               Pose.from_array([float(v) for v in tok[5:12]])))
            elif head == "patch":
                patches.append((int(tok[1]), int(tok[2]), float(tok[3]), int(tok[4]),
                                np.array([float(v) for v in tok[5:]]).reshape(-1, 2)))
            elif head == "edge":
                kind = tok[4]
                if kind not in _KIND_CODE:
                    raise ValueError(f"unknown edge kind {kind!r}")
                conf = np.array([float(tok[5]), float(tok[6])])
                if np.any(conf < 0) or np.any(conf > 1):
                    raise ValueError(f"confidence must lie in [0, 1], got {conf}")
                src, dst = int(tok[1]), int(tok[3])
                if kind == LOOP and src == dst:
                    raise ValueError("loop edges must connect distinct frames")
                edges.append((src, int(tok[2]), dst, kind, conf,
                              np.array([float(v) for v in tok[7:]]).reshape(-1, 2)))
            else:
                extras.append((ln, tok))
        except (ValueError, IndexError) as exc:
            raise ParseError(f"bad {head!r} record: {exc}", path, ln) from exc
    if intr is None:
        raise ParseError("missing intrinsics record", path)

    g = PatchGraph(intr, p)
    m = p * p
    frames.sort(key=lambda r: r[0])
    per_frame = {r[0]: [] for r in frames}
    for fid, idx, d, lm, grid in patches:
        if fid not in per_frame:
            raise ParseError(f"patch of unknown frame {fid}", path)
        if grid.shape[0] != m:
            raise ValueError(f"patch size {int(round(np.sqrt(grid.shape[0])))} != graph "
                             f"patch size {p}")
        per_frame[fid].append((idx, d, lm, grid))
    for fid, ts, kf, feat, pose in frames:
        rows = sorted(per_frame[fid], key=lambda r: r[0])
        grids = np.stack([r[3] for r in rows]) if rows else np.zeros((0, m, 2))
        got = g.add_frame_arrays(pose.q, pose.t, ts, grids,
                                 np.array([r[1] for r in rows], dtype=float),
                                 np.array([r[2] for r in rows], dtype=np.int64), kf)
        if got != fid:
            raise ParseError(f"non-contiguous frame ids near frame {fid}", path)
        g._feat.view[fid] = feat
    if edges:
        for i, k, j, *_ in edges:
            g._check_edge_indices(i, k, j)
        n = len(edges)
        g._src.extend(np.array([e[0] for e in edges]))
        g._pat.extend(np.array([e[1] for e in edges]))
        g._dst.extend(np.array([e[2] for e in edges]))
        g._tgt.extend(np.stack([e[5] for e in edges]).reshape(n, -1, 2))
        g._conf.extend(np.stack([e[4] for e in edges]))
        g._kind.extend(np.array([_KIND_CODE[e[3]] for e in edges], dtype=np.uint8))
    return g, extras


def read_graph(path) -> PatchGraph:
    with open(path) as fh:
        g, _ = parse_graph_lines(fh, str(path))
    return g
