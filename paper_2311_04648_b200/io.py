"""Frame output of the drop-in (grainforge/io.py:120-196): sphere CSV and
mesh VTK frames written from device snapshots -- the per-sphere columns are
assembled on the device in one pass (gf_sphere_frame) and come back as one
array; no owner-state download.  The text layout is the reference's:
columns in the declared content order, full-precision %.17g numbers, so a
frame of the same state is byte-identical."""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import ValidationError

_CONTENT_COLUMNS = {
    "XYZ": ("x", "y", "z"),
    "ABSV": ("absv",),
    "FAMILY": ("family",),
    "VEL": ("vx", "vy", "vz"),
}
_FIELDS = {"XYZ": (0, 1, 2), "ABSV": (3,), "FAMILY": (4,), "VEL": (5, 6, 7)}


def _fmt(x: float) -> str:
    return format(float(x), ".17g")


def sphere_frame(sim) -> np.ndarray:
    """(n_spheres, 8) float64 in the reference's sphere order: centre xyz,
    |v|, family, v xyz of the owner -- one device pass, one copy."""
    n = int(sim._sph_geom.size)
    out = np.zeros((n, 8), np.float64)
    if n:
        sim._push_host()
        dev = np.zeros((n, 8), np.float64)
        sim._ctx.call("gf_sphere_frame", _lib.ptr(dev))
        out[sim._sph_d2u] = dev
    return out


def write_sphere_csv(sim, path, content=("XYZ", "ABSV")) -> None:
    """One row per component sphere (io.py:132-166)."""
    for item in content:
        if item not in _CONTENT_COLUMNS:
            raise ValidationError(f"unknown output content {item!r}")
    fr = sphere_frame(sim)
    header = ",".join(col for item in content for col in _CONTENT_COLUMNS[item])
    lines = [header]
    for row in fr:
        cols = []
        for item in content:
            if item == "FAMILY":
                cols.append(str(int(row[4])))
            else:
                cols += [_fmt(row[f]) for f in _FIELDS[item]]
        lines.append(",".join(cols))
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


def write_mesh_vtk(sim, path, owners=None) -> None:
    """Legacy-ASCII unstructured grid of all (or the given) mesh owners in
    their current world pose, three points per facet (io.py:169-196); the
    world triangles come from the device."""
    from .core import GEOM_TRIANGLE
    s = sim.store
    tri = np.nonzero(s.geom_kind[: s.n_geoms] == GEOM_TRIANGLE)[0]
    if owners is not None:
        tri = tri[np.isin(s.geom_owner[tri], np.asarray(owners))]
    slot = sim._geom_slot[tri] if tri.size else np.zeros(0, dtype=np.int64)
    world = sim._tri_world[slot] if tri.size else np.zeros((0, 9))
    n_pts = 3 * world.shape[0]
    lines = ["# vtk DataFile Version 2.0", "grainforge mesh", "ASCII", "DATASET UNSTRUCTURED_GRID",
             f"POINTS {n_pts} double"]
    for row in world:
        for v in range(3):
            lines.append(f"{_fmt(row[3 * v])} {_fmt(row[3 * v + 1])} {_fmt(row[3 * v + 2])}")
    m = world.shape[0]
    lines.append(f"CELLS {m} {4 * m}")
    for k in range(m):
        lines.append(f"3 {3 * k} {3 * k + 1} {3 * k + 2}")
    lines.append(f"CELL_TYPES {m}")
    lines.extend(["5"] * m)
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")
