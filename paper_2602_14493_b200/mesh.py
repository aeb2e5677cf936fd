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


# ---------------------------------------------------------------------------
# File formats on either side of the path (reference mesh.py:161-421): ASCII
# PLY writer; OBJ and PLY (ascii / binary_little_endian) readers with fan
# triangulation.  Host-side I/O, not part of the device path.
# ---------------------------------------------------------------------------

class MeshParseError(MeshError):
    """Malformed mesh file (mesh.py:22-28): message prefixed with path:line."""

    def __init__(self, path, line, message):
        super().__init__(f"{path}:{line}: {message}")
        self.path, self.line = path, line


_PLY_TYPES = {"char": "i1", "int8": "i1", "uchar": "u1", "uint8": "u1", "short": "i2", "int16": "i2",
              "ushort": "u2", "uint16": "u2", "int": "i4", "int32": "i4", "uint": "u4", "uint32": "u4",
              "float": "f4", "float32": "f4", "double": "f8", "float64": "f8"}


def save_mesh(mesh: TriangleMesh, path) -> None:
    """ASCII PLY, double positions and colours printed with %.17g so a
    reload reproduces the mesh exactly (mesh.py:395-421)."""
    head = ["ply", "format ascii 1.0", "comment meshsplat", f"element vertex {mesh.num_vertices}",
            "property double x", "property double y", "property double z",
            "property double red", "property double green", "property double blue",
            f"element face {mesh.num_facets}", "property list uchar int vertex_indices", "end_header"]
    vc = np.concatenate([mesh.vertices, mesh.colors], axis=1)
    body = ["%.17g %.17g %.17g %.17g %.17g %.17g" % tuple(r) for r in vc.tolist()]
    body += ["3 %d %d %d" % tuple(f) for f in np.asarray(mesh.facets).tolist()]
    with open(path, "w") as fh:
        fh.write("\n".join(head + body) + "\n")


def _fan(idx, nv, path, where):
    for i in idx:
        if not 0 <= i < nv:
            raise MeshParseError(path, where, f"vertex index {i} out of range [0, {nv})")
    if len(idx) < 3:
        raise MeshParseError(path, where, "face with fewer than 3 vertices")
    return [(idx[0], idx[k], idx[k + 1]) for k in range(1, len(idx) - 1)]


def _read_obj(path) -> TriangleMesh:
    verts, cols, tris, colored = [], [], [], False
    with open(path, errors="replace") as fh:
        for n, raw in enumerate(fh, start=1):
            tok = raw.split()
            if not tok or tok[0].startswith("#"):
                continue
            if tok[0] == "v":
                try:
                    x = [float(t) for t in tok[1:]]
                except ValueError:
                    raise MeshParseError(path, n, f"bad vertex line: {raw.strip()!r}") from None
                if len(x) < 3:
                    raise MeshParseError(path, n, "vertex line needs at least 3 coordinates")
                verts.append(x[:3])
                if len(x) >= 6:
                    cols.append(x[3:6] if len(x) > 6 else x[-3:])
                    colored = True
                else:
                    cols.append([GRAY] * 3)
            elif tok[0] == "f":
                idx = []
                for t in tok[1:]:
                    try:
                        i = int(t.split("/")[0])
                    except ValueError:
                        raise MeshParseError(path, n, f"bad face token {t!r}") from None
                    if i == 0:
                        raise MeshParseError(path, n, "OBJ face indices are 1-based; got 0")
                    idx.append(i - 1 if i > 0 else len(verts) + i)
                tris.extend(_fan(idx, len(verts), path, n))
    try:
        return TriangleMesh(np.asarray(verts, np.float64).reshape(-1, 3), tris,
                            np.clip(cols, 0.0, 1.0) if colored else None)
    except MeshError as e:
        raise MeshParseError(path, 0, str(e)) from None


def _read_ply(path) -> TriangleMesh:
    with open(path, "rb") as fh:
        if fh.readline().strip() != b"ply":
            raise MeshParseError(path, 1, "not a PLY file (missing 'ply' magic)")
        fmt, elems, n = None, [], 1
        while True:
            raw = fh.readline()
            n += 1
            if not raw:
                raise MeshParseError(path, n, "unexpected EOF in header")
            tok = raw.decode("ascii", errors="replace").split()
            if not tok or tok[0] in ("comment", "obj_info"):
                continue
            if tok[0] == "format":
                fmt = tok[1]
                if fmt not in ("ascii", "binary_little_endian"):
                    raise MeshParseError(path, n, f"unsupported PLY format {fmt!r}")
            elif tok[0] == "element":
                elems.append((tok[1], int(tok[2]), []))
            elif tok[0] == "property":
                if not elems:
                    raise MeshParseError(path, n, "property before any element")
                if tok[1] == "list":
                    if tok[2] not in _PLY_TYPES or tok[3] not in _PLY_TYPES:
                        raise MeshParseError(path, n, f"unknown list types {tok[2]}/{tok[3]}")
                    elems[-1][2].append((tok[4], ("list", _PLY_TYPES[tok[2]], _PLY_TYPES[tok[3]])))
                else:
                    if tok[1] not in _PLY_TYPES:
                        raise MeshParseError(path, n, f"unknown property type {tok[1]!r}")
                    elems[-1][2].append((tok[2], _PLY_TYPES[tok[1]]))
            elif tok[0] == "end_header":
                break
            else:
                raise MeshParseError(path, n, f"unknown header keyword {tok[0]!r}")
        if fmt is None:
            raise MeshParseError(path, n, "missing 'format' line")
        data = {}
        for name, count, props in elems:
            if fmt == "ascii":
                cols = [[] for _ in props]
                for _ in range(count):
                    raw = fh.readline()
                    n += 1
                    if not raw:
                        raise MeshParseError(path, n, f"unexpected EOF in element {name!r}")
                    tok, k = raw.split(), 0
                    try:
                        for ci, (_, kind) in enumerate(props):
                            if isinstance(kind, tuple):
                                m = int(tok[k])
                                vals = [float(t) for t in tok[k + 1:k + 1 + m]]
                                if len(vals) != m:
                                    raise IndexError
                                cols[ci].append(np.array(vals))
                                k += 1 + m
                            else:
                                cols[ci].append(float(tok[k]))
                                k += 1
                    except (IndexError, ValueError):
                        raise MeshParseError(path, n, f"malformed {name!r} row") from None
                data[name] = (props, [c if isinstance(props[i][1], tuple) else np.asarray(c, np.float64)
                                      for i, c in enumerate(cols)])
            elif not any(isinstance(p[1], tuple) for p in props):
                dt = np.dtype([(f"f{i}", "<" + kind) for i, (_, kind) in enumerate(props)])
                buf = fh.read(dt.itemsize * count)
                if len(buf) != dt.itemsize * count:
                    raise MeshParseError(path, n, f"truncated binary element {name!r}")
                rec = np.frombuffer(buf, dtype=dt)
                data[name] = (props, [rec[f"f{i}"].astype(np.float64) for i in range(len(props))])
            else:
                if len(props) != 1:
                    raise MeshParseError(path, n, f"mixed list/scalar element {name!r} unsupported")
                cdt, idt = np.dtype("<" + props[0][1][1]), np.dtype("<" + props[0][1][2])
                lists = []
                for row in range(count):
                    cb = fh.read(cdt.itemsize)
                    if len(cb) != cdt.itemsize:
                        raise MeshParseError(path, n, f"truncated {name!r} at row {row}")
                    m = int(np.frombuffer(cb, cdt)[0])
                    ib = fh.read(idt.itemsize * m)
                    if len(ib) != idt.itemsize * m:
                        raise MeshParseError(path, n, f"truncated {name!r} at row {row}")
                    lists.append(np.frombuffer(ib, idt).astype(np.int64))
                data[name] = (props, [lists])
    if "vertex" not in data:
        raise MeshParseError(path, 0, "PLY without a vertex element")
    props, cols = data["vertex"]
    names = [p[0] for p in props]
    for c in "xyz":
        if c not in names:
            raise MeshParseError(path, 0, f"vertex element lacks property {c!r}")
    verts = np.stack([cols[names.index(c)] for c in "xyz"], axis=1)
    colors = None
    if all(c in names for c in ("red", "green", "blue")):
        ch = [cols[names.index(c)] / (255.0 if props[names.index(c)][1] == "u1" else 1.0)
              for c in ("red", "green", "blue")]
        colors = np.clip(np.stack(ch, axis=1), 0.0, 1.0)
    tris = []
    if "face" in data:
        props, cols = data["face"]
        names = [p[0] for p in props]
        key = next((k for k in ("vertex_indices", "vertex_index") if k in names), None)
        if key is None:
            raise MeshParseError(path, 0, "face element lacks vertex_indices")
        for fi, idx in enumerate(cols[names.index(key)]):
            tris.extend(_fan([int(i) for i in idx], len(verts), path, f"face {fi}"))
    try:
        return TriangleMesh(verts, tris, colors)
    except MeshError as e:
        raise MeshParseError(path, 0, str(e)) from None


def load_mesh(path) -> TriangleMesh:
    """OBJ or PLY by extension (mesh.py:177-199)."""
    import os
    ext = os.path.splitext(str(path))[1].lower()
    if ext == ".obj":
        return _read_obj(path)
    if ext == ".ply":
        return _read_ply(path)
    raise MeshParseError(path, 0, f"unsupported mesh extension {ext!r}")
