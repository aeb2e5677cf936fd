"""Triangle mesh container and synthetic mesh generators.

`TriangleMesh` mirrors the reference's immutable container and its
validation (`pkg/src/meshsplat/mesh.py:46-130`).  On the device a mesh is
SoA-free AoS: `pos[V*3]` f32/f64, `col[V*3]`, `faces[F*3]` int32 (the
`GmrMesh` view of `include/gmr.h`).  The generators build the benchmark
configurations of BASELINE.json: `make_icosphere` (reference
`mesh.py:463-505`, same vertex/face order) and the class-I geodesic
displaced sphere of SURVEY §8d (configs 3-4).
"""

from __future__ import annotations

from functools import cached_property

import numpy as np

GRAY = 0.5
DEGENERATE_AREA_EPS = 1e-12


class MeshError(ValueError):
    """Invalid mesh data (mesh.py:18-19)."""


def _float_rows(values, name):
    arr = np.asarray(values, dtype=np.float64)
    if arr.size == 0:
        arr = arr.reshape(0, 3)
    if arr.ndim != 2 or arr.shape[1] != 3:
        raise MeshError(f"{name} must have shape (n, 3), got {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise MeshError(f"{name} contains non-finite values")
    return arr


class TriangleMesh:
    """Immutable V x 3 vertices, F x 3 facets, V x 3 colours in [0, 1]."""

    def __init__(self, vertices, facets, colors=None):
        verts = _float_rows(vertices, "vertices")
        f = np.asarray(facets, dtype=np.int64)
        if f.size == 0:
            f = f.reshape(0, 3)
        if f.ndim != 2 or f.shape[1] != 3:
            raise MeshError(f"facets must have shape (m, 3), got {f.shape}")
        n = len(verts)
        if f.size and (f.min() < 0 or f.max() >= n):
            bad = int(np.argmax((f < 0) | (f >= n)).item() // 3)
            raise MeshError(f"facet {bad} references a vertex index outside [0, {n})")
        if f.size:
            rep = (f[:, 0] == f[:, 1]) | (f[:, 1] == f[:, 2]) | (f[:, 0] == f[:, 2])
            if rep.any():
                raise MeshError(f"facet {int(np.argmax(rep))} has repeated vertex indices")
        col = np.full((n, 3), GRAY) if colors is None else colors
        col = _float_rows(col, "colors")
        if len(col) != n:
            raise MeshError(f"colors length {len(col)} != vertex count {n}")
        if col.size and (col.min() < -1e-9 or col.max() > 1 + 1e-9):
            raise MeshError("colors must lie in [0, 1]")
        col = np.clip(col, 0.0, 1.0)
        for a in (verts, f, col):
            a.setflags(write=False)
        self.vertices, self.facets, self.colors = verts, f, col

    @property
    def num_vertices(self):
        return len(self.vertices)

    @property
    def num_facets(self):
        return len(self.facets)

    @cached_property
    def edges(self):
        """Unique undirected edges, smaller index first, lexsorted (mesh.py:96-106)."""
        if self.num_facets == 0:
            e = np.zeros((0, 2), dtype=np.int64)
        else:
            e = np.unique(np.sort(self.facets[:, [0, 1, 1, 2, 2, 0]].reshape(-1, 2), axis=1), axis=0)
        e.setflags(write=False)
        return e

    def with_vertices(self, vertices, colors=None):
        return TriangleMesh(vertices, self.facets, self.colors if colors is None else colors)


def make_icosphere(target_facets: int, radius: float = 1.0) -> TriangleMesh:
    """Smallest icosahedron subdivision with >= target_facets facets; same
    construction order as the reference (mesh.py:463-505) so vertex and
    facet indices coincide."""
    if target_facets < 20:
        raise MeshError("target_facets must be >= 20")
    level = 0
    while 20 * 4 ** level < target_facets:
        level += 1
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    base = np.array([(-1, phi, 0), (1, phi, 0), (-1, -phi, 0), (1, -phi, 0),
                     (0, -1, phi), (0, 1, phi), (0, -1, -phi), (0, 1, -phi),
                     (phi, 0, -1), (phi, 0, 1), (-phi, 0, -1), (-phi, 0, 1)], dtype=np.float64)
    base /= np.linalg.norm(base[0])
    tris = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
            (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
            (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
            (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    pts = list(base)
    for _ in range(level):
        mids = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            idx = mids.get(key)
            if idx is None:
                m = pts[a] + pts[b]
                pts.append(m / np.linalg.norm(m))
                idx = mids[key] = len(pts) - 1
            return idx

        nxt = []
        for a, b, c in tris:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nxt += [(a, ab, ca), (ab, b, bc), (ca, bc, c), (ab, bc, ca)]
        tris = nxt
    return TriangleMesh(np.asarray(pts) * radius, tris)


def _icosahedron():
    m = make_icosphere(20)
    return np.asarray(m.vertices), np.asarray(m.facets)


def make_geodesic_sphere(frequency: int, amplitude: float = 0.05, seed: int = 0,
                         colors: bool = True) -> TriangleMesh:
    """Class-I geodesic sphere of the given frequency n (20 n^2 facets,
    10 n^2 + 2 vertices), radially displaced by
    r(v) = 1 + amplitude * sum_{i<6} sin(3 d_i . v) / 6 with d_i ~ N(0, I)
    drawn from `default_rng(seed)`.  Vertex colours
    are U[0.1, 0.9] from `default_rng(seed + 1)`.  n = 158 gives 499,280
    facets; n = 316 gives 1,997,120."""
    n = int(frequency)
    if n < 1:
        raise MeshError("frequency must be >= 1")
    cv, cf = _icosahedron()
    # barycentric lattice (i, j, k), i + j + k = n
    ii, jj = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    ok = ii + jj <= n
    gi, gj = ii[ok], jj[ok]
    gk = n - gi - gj
    lut = -np.ones((n + 1, n + 1), dtype=np.int64)
    lut[gi, gj] = np.arange(len(gi))
    npts = len(gi)
    # canonical key per lattice point of every face: (vertex id, weight)
    # pairs sorted by vertex id so shared edge / corner points coincide
    vid = cf[:, None, :].repeat(npts, axis=1)                    # (20, P, 3)
    wt = np.stack([gk, gi, gj], axis=1)[None].repeat(20, axis=0)  # weights of corners a, b, c
    raw = np.where(wt > 0, vid * (n + 1) + wt, -1)
    order = np.argsort(raw, axis=2, kind="stable")
    vid_s = np.take_along_axis(vid, order, axis=2)
    wt_s = np.take_along_axis(wt, order, axis=2)
    key = np.take_along_axis(raw, order, axis=2).reshape(-1, 3)
    uniq, first, inverse = np.unique(key, axis=0, return_index=True, return_inverse=True)
    inverse = inverse.reshape(20, npts)
    flat_vid = vid_s.reshape(-1, 3)[first]
    flat_wt = wt_s.reshape(-1, 3)[first].astype(np.float64)
    p = (flat_wt[:, 0:1] * cv[flat_vid[:, 0]] + flat_wt[:, 1:2] * cv[flat_vid[:, 1]]
         + flat_wt[:, 2:3] * cv[flat_vid[:, 2]])
    unit = p / np.linalg.norm(p, axis=1, keepdims=True)
    # small triangles of each face, orientation of (a, b, c)
    ui, uj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    up = ui + uj <= n - 1
    ui, uj = ui[up], uj[up]
    tri_up = np.stack([lut[ui, uj], lut[ui + 1, uj], lut[ui, uj + 1]], axis=1)
    dn = ui + uj <= n - 2
    di, dj = ui[dn], uj[dn]
    tri_dn = np.stack([lut[di + 1, dj], lut[di + 1, dj + 1], lut[di, dj + 1]], axis=1)
    local = np.concatenate([tri_up, tri_dn])                      # (n^2, 3) lattice ids
    facets = inverse[np.arange(20)[:, None, None], local[None]].reshape(-1, 3)
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(6, 3))
    r = 1.0 + amplitude * np.sin(3.0 * unit @ d.T).sum(axis=1) / 6.0
    verts = unit * r[:, None]
    col = np.random.default_rng(seed + 1).uniform(0.1, 0.9, size=(len(verts), 3)) if colors else None
    return TriangleMesh(verts, facets, col)


def seeded_colors(num_vertices: int, seed: int = 0) -> np.ndarray:
    """Vertex colours U[0.1, 0.9] (SURVEY §8d shared settings)."""
    return np.random.default_rng(seed).uniform(0.1, 0.9, size=(num_vertices, 3))


def make_grid_cube(divisions: int = 8, half_extent: float = 1.0, position_colors: bool = False) -> TriangleMesh:
    """Axis-aligned cube, each face a divisions x divisions grid of quads
    (two triangles each), outward winding; same vertex/facet order as the
    reference (mesh.py:508-550)."""
    if divisions < 1:
        raise MeshError("divisions must be >= 1")
    pts, tris, index = [], [], {}

    def vid(p):
        key = tuple(np.round(p, 12))
        if key not in index:
            index[key] = len(pts)
            pts.append(np.asarray(p, dtype=np.float64))
        return index[key]

    h = half_extent
    lin = np.linspace(-h, h, divisions + 1)
    for axis in range(3):
        for sign in (-1.0, 1.0):
            ua, va = [a for a in range(3) if a != axis]
            for i in range(divisions):
                for j in range(divisions):
                    quad = []
                    for du, dv in ((0, 0), (1, 0), (1, 1), (0, 1)):
                        p = np.zeros(3)
                        p[axis] = sign * h
                        p[ua] = lin[i + du]
                        p[va] = lin[j + dv]
                        quad.append(vid(p))
                    a, b, c, d = quad
                    if (sign > 0) ^ (axis == 1):
                        tris += [(a, b, c), (a, c, d)]
                    else:
                        tris += [(a, c, b), (a, d, c)]
    verts = np.asarray(pts)
    col = np.clip((verts / h + 1.0) / 2.0, 0.0, 1.0) if position_colors else None
    return TriangleMesh(verts, tris, col)


def _diameter(points) -> float:
    pts = np.asarray(points, dtype=np.float64)
    if len(pts) > 1024:
        try:
            from scipy.spatial import ConvexHull
            pts = pts[ConvexHull(pts).vertices]
        except Exception:
            pass
    best = 0.0
    block = max(1, int(2 ** 22 // max(len(pts), 1)))
    for s in range(0, len(pts), block):
        d2 = ((pts[s:s + block, None, :] - pts[None, :, :]) ** 2).sum(axis=2)
        best = max(best, float(d2.max()))
    return float(np.sqrt(best))


def normalize_mesh(mesh: TriangleMesh):
    """Centre on the bounding-box centre, scale the diameter to 2
    (reference mesh.py:428-456).  Returns (mesh, (center, scale))."""
    if mesh.num_vertices < 2:
        raise MeshError("need at least 2 vertices to normalize")
    d = _diameter(mesh.vertices)
    if d < 1e-12:
        raise MeshError("all vertices coincide; cannot normalize")
    center = 0.5 * (mesh.vertices.min(axis=0) + mesh.vertices.max(axis=0))
    scale = 2.0 / d
    return mesh.with_vertices(scale * (mesh.vertices - center)), (center, scale)


def make_grid_cube_normalized(divisions: int = 4) -> TriangleMesh:
    """Config 5 target: normalize_mesh(make_grid_cube(divisions, position_colors=True))."""
    return normalize_mesh(make_grid_cube(divisions, position_colors=True))[0]


def mesh_graph(facets, num_vertices):
    """Edges, vertex->(edge, endpoint) CSR in np.add.at order and the sorted
    neighbour CSR (reference mesh.py:96-126, losses.py:95-96), int32."""
    f = np.asarray(facets)
    e = (np.unique(np.sort(f[:, [0, 1, 1, 2, 2, 0]].reshape(-1, 2), axis=1), axis=0)
         if len(f) else np.zeros((0, 2), np.int64))
    E = len(e)
    keys = np.concatenate([e[:, 1], e[:, 0]])
    slots = np.concatenate([2 * np.arange(E) + 1, 2 * np.arange(E)])
    order = np.argsort(keys, kind="stable")
    ve_slot = slots[order]
    ve_ptr = np.concatenate([[0], np.cumsum(np.bincount(keys, minlength=num_vertices))])
    both = np.concatenate([e, e[:, ::-1]]) if E else np.zeros((0, 2), np.int64)
    both = both[np.lexsort((both[:, 1], both[:, 0]))]
    adj_ptr = np.concatenate([[0], np.cumsum(np.bincount(both[:, 0], minlength=num_vertices))])
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    return dict(edges=i32(e.reshape(-1, 2)), ve_ptr=i32(ve_ptr), ve_slot=i32(ve_slot), adj_ptr=i32(adj_ptr),
                adj=i32(both[:, 1]))
