"""Contact arrays, margins and the detection entry points of the drop-in
(mirrors grainforge/broadphase.py: compute_margin :24, MarginPolicy :35,
ContactArray :48, merge_history :110, DetectionSnapshot :139,
detect_contacts :202).

detect_contacts and merge_history execute on the device (csrc/gf_kt.cu); the
pair list is bit-identical to the reference's for the same snapshot.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import ValidationError
from .types import REAL

CONTACT_SS = 0
CONTACT_ST = 1
CONTACT_SA = 2

# Device keys hold 31-bit geometry ids (the reference's key budget is 24 bits,
# broadphase.py:21); the (kind, a, b) order is the same.
_KEY_GEOM_BITS = 31


def compute_margin(v_max: float, h: float, n_max: int) -> float:
    if v_max <= 0.0 or h <= 0.0 or n_max <= 0:
        raise ValidationError(f"margin inputs must be positive (v_max={v_max}, h={h}, n_max={n_max})")
    return 2.0 * v_max * h * n_max


@dataclass
class MarginPolicy:
    v_max: float
    h: float
    n_max: int
    added: float = 0.0

    @property
    def margin(self) -> float:
        return compute_margin(self.v_max, self.h, self.n_max) + self.added


class ContactArray:
    """Candidate pairs in canonical (kind, geom_a, geom_b) order plus named
    float32 wildcard columns (host container; broadphase.py:48-107)."""

    def __init__(self, kind=None, geom_a=None, geom_b=None, wildcards=None):
        self.kind = np.asarray([] if kind is None else kind, dtype=np.uint8)
        self.geom_a = np.asarray([] if geom_a is None else geom_a, dtype=np.int64)
        self.geom_b = np.asarray([] if geom_b is None else geom_b, dtype=np.int64)
        self.wildcards: dict = {}
        for name, values in (wildcards or {}).items():
            arr = np.asarray(values, dtype=REAL)
            if arr.shape[0] != self.size:
                raise ValidationError(f"wildcard {name!r} length {arr.shape[0]} != pair count {self.size}")
            self.wildcards[name] = arr

    @property
    def size(self) -> int:
        return int(self.geom_a.shape[0])

    def __len__(self):
        return self.size

    def sort_keys(self) -> np.ndarray:
        lim = 1 << _KEY_GEOM_BITS
        if np.any(self.geom_a >= lim) or np.any(self.geom_b >= lim):
            raise ValidationError("geometry ids exceed the sort-key budget")
        return ((self.kind.astype(np.uint64) << np.uint64(2 * _KEY_GEOM_BITS))
                | (self.geom_a.astype(np.uint64) << np.uint64(_KEY_GEOM_BITS))
                | self.geom_b.astype(np.uint64))

    def canonicalize(self) -> "ContactArray":
        order = np.argsort(self.sort_keys(), kind="stable")
        out = ContactArray(self.kind[order], self.geom_a[order], self.geom_b[order])
        out.wildcards = {k: v[order] for k, v in self.wildcards.items()}
        return out

    def ensure_wildcards(self, names) -> None:
        for name in names:
            self.wildcards.setdefault(name, np.zeros(self.size, dtype=REAL))

    def select(self, keep_mask) -> "ContactArray":
        out = ContactArray(self.kind[keep_mask], self.geom_a[keep_mask], self.geom_b[keep_mask])
        out.wildcards = {k: v[keep_mask] for k, v in self.wildcards.items()}
        return out


@dataclass
class DetectionSnapshot:
    sph_center: np.ndarray
    sph_radius: np.ndarray
    sph_geom: np.ndarray
    sph_owner: np.ndarray
    sph_family: np.ndarray
    tri_world: np.ndarray
    tri_geom: np.ndarray
    tri_owner: np.ndarray
    tri_family: np.ndarray
    ana_world: np.ndarray
    ana_kind: np.ndarray
    ana_geom: np.ndarray
    ana_owner: np.ndarray
    ana_family: np.ndarray
    mask: np.ndarray
    stamp: int = 0


_UTIL_CTX = {}


def _util_ctx(device: int = 0) -> _lib.Context:
    ctx = _UTIL_CTX.get(device)
    if ctx is None:
        ctx = _UTIL_CTX[device] = _lib.Context(device)
    return ctx


def detect_contacts_raw(snapshot: DetectionSnapshot, margin: float, bin_size=None, device: int = 0):
    """Device detection on a snapshot; returns (kind, slot_a, slot_b, glo,
    inv_bin, nb) with slots in each kind's own numbering."""
    if margin < 0.0:
        raise ValidationError(f"margin must be non-negative, got {margin}")
    s = snapshot
    c = _lib.carr(s.sph_center, np.float64).reshape(-1, 3)
    rad = _lib.carr(s.sph_radius, np.float32)
    m = c.shape[0]
    r_max = float(rad.max()) if m else 0.0
    if bin_size is not None and bin_size < 2.0 * (r_max + margin):
        raise ValidationError(f"bin_size {bin_size} below max enlarged sphere diameter "
                              f"{2.0 * (r_max + margin)}")
    tri = _lib.carr(s.tri_world, np.float64).reshape(-1, 9)
    ana = _lib.carr(s.ana_world, np.float64).reshape(-1, 8)
    grid = np.zeros(4, np.float64)
    nb = np.zeros(3, np.int64)
    n_out = C.c_int64(0)
    ctx = _util_ctx(device)
    keep = [c, rad, _lib.carr(s.sph_owner, np.int64), _lib.carr(s.sph_family, np.uint8), tri,
            _lib.carr(s.tri_owner, np.int64), _lib.carr(s.tri_family, np.uint8), ana,
            _lib.carr(s.ana_kind, np.uint8), _lib.carr(s.ana_owner, np.int64),
            _lib.carr(s.ana_family, np.uint8), _lib.carr(s.mask, np.uint8).reshape(-1)]
    P = _lib.ptr
    ctx.call("gf_detect_snapshot", C.c_int64(m), P(keep[0]), P(keep[1]), P(keep[2]), P(keep[3]),
             C.c_int64(tri.shape[0]), P(keep[4]), P(keep[5]), P(keep[6]),
             C.c_int64(ana.shape[0]), P(keep[7]), P(keep[8]), P(keep[9]), P(keep[10]),
             P(keep[11]), C.c_double(margin), C.c_double(-1.0 if bin_size is None else bin_size),
             P(grid), P(nb), C.byref(n_out))
    n = int(n_out.value)
    kind = np.zeros(n, np.uint8)
    sa = np.zeros(n, np.int64)
    sb = np.zeros(n, np.int64)
    if n:
        ctx.call("gf_get_acs", C.c_int(1), P(kind), P(sa), P(sb), None)
    return kind, sa, sb, grid[:3].copy(), float(grid[3]), nb


def detect_contacts(snapshot: DetectionSnapshot, margin: float, bin_size=None) -> ContactArray:
    """Exactly the reference's pairs (broadphase.py:202-288), canonical order."""
    kind, sa, sb, _, _, _ = detect_contacts_raw(snapshot, margin, bin_size)
    s = snapshot
    ga = np.asarray(s.sph_geom, np.int64)[sa] if kind.size else np.zeros(0, np.int64)
    tabs = (np.asarray(s.sph_geom, np.int64), np.asarray(s.tri_geom, np.int64),
            np.asarray(s.ana_geom, np.int64))
    gb = np.zeros(kind.shape[0], np.int64)
    for k in range(3):
        sel = kind == k
        if sel.any():
            gb[sel] = tabs[k][sb[sel]]
    arr = ContactArray(kind, ga, gb)
    # slots are monotone in geometry id for engine snapshots; sort anyway so
    # arbitrary snapshots come back canonical too
    return arr.canonicalize()


def merge_history(old: ContactArray, new_pairs: ContactArray) -> ContactArray:
    """History-preserving merge on the device (broadphase.py:110-135)."""
    out = ContactArray(new_pairs.kind.copy(), new_pairs.geom_a.copy(), new_pairs.geom_b.copy())
    names = list(dict.fromkeys(list(old.wildcards) + list(new_pairs.wildcards)))
    if not names:
        return out
    if old.size == 0 or out.size == 0:
        for name in names:
            out.wildcards[name] = np.zeros(out.size, dtype=REAL)
        return out
    old_w = np.stack([old.wildcards.get(n, np.zeros(old.size, REAL)) for n in names], axis=1)
    old_w = np.ascontiguousarray(old_w, dtype=np.float32)
    res = np.zeros((out.size, len(names)), np.float32)
    ctx = _util_ctx(0)
    P = _lib.ptr
    ok = _lib.carr(old.kind, np.uint8), _lib.carr(old.geom_a, np.int64), _lib.carr(old.geom_b, np.int64)
    nk = _lib.carr(out.kind, np.uint8), _lib.carr(out.geom_a, np.int64), _lib.carr(out.geom_b, np.int64)
    ctx.call("gf_merge_history", C.c_int64(old.size), P(ok[0]), P(ok[1]), P(ok[2]), P(old_w),
             C.c_int64(out.size), P(nk[0]), P(nk[1]), P(nk[2]), C.c_int(len(names)), P(res))
    for i, name in enumerate(names):
        out.wildcards[name] = res[:, i].copy()
    return out


def build_bins(centers, radii, bin_size, margin: float = 0.0):
    """Uniform-grid CSR of the margin-enlarged sphere boxes (broadphase.py:
    303-323; exposed for tests -- detection itself enumerates centre cells,
    csrc/gf_kt.cu).  The per-sphere bin ranges come from the device
    (gf_bin_ranges on the reference grid); the CSR keeps the reference's
    stable sphere order within a bin.  Returns (grid_lo, inv_bin_size,
    bins_per_axis, starts, entries)."""
    centers = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
    radii = np.asarray(radii, dtype=REAL).reshape(-1)
    r_max = float(radii.max()) if radii.size else 0.0
    min_bin = 2.0 * (r_max + margin)
    if bin_size < min_bin:
        raise ValidationError(f"bin_size {bin_size} below max enlarged sphere diameter {min_bin}")
    m = centers.shape[0]
    snap = DetectionSnapshot(
        sph_center=centers, sph_radius=radii, sph_geom=np.arange(m, dtype=np.int64),
        sph_owner=np.arange(m, dtype=np.int64), sph_family=np.zeros(m, np.uint8),
        tri_world=np.zeros((0, 9)), tri_geom=np.zeros(0, np.int64), tri_owner=np.zeros(0, np.int64),
        tri_family=np.zeros(0, np.uint8), ana_world=np.zeros((0, 8)), ana_kind=np.zeros(0, np.uint8),
        ana_geom=np.zeros(0, np.int64), ana_owner=np.zeros(0, np.int64), ana_family=np.zeros(0, np.uint8),
        mask=np.ones((256, 256), dtype=bool))
    _, _, _, glo, inv, nb = detect_contacts_raw(snap, margin, bin_size)
    ranges = np.zeros((m, 6), np.int64)
    if m:
        _util_ctx(0).call("gf_bin_ranges", C.c_double(margin), _lib.ptr(ranges))
    # (bin, sphere) registrations, stable in sphere order within a bin (_kernels.py:270-283)
    bins, owners = [], []
    for i in range(m):
        xs = np.arange(ranges[i, 0], ranges[i, 1] + 1)
        ys = np.arange(ranges[i, 2], ranges[i, 3] + 1)
        zs = np.arange(ranges[i, 4], ranges[i, 5] + 1)
        b = ((zs[:, None, None] * nb[1] + ys[None, :, None]) * nb[0] + xs[None, None, :]).reshape(-1)
        bins.append(b)
        owners.append(np.full(b.size, i, np.int64))
    nbins = int(nb[0] * nb[1] * nb[2])
    b = np.concatenate(bins) if bins else np.zeros(0, np.int64)
    o = np.concatenate(owners) if owners else np.zeros(0, np.int64)
    order = np.argsort(b, kind="stable")
    starts = np.zeros(nbins + 1, np.int64)
    np.cumsum(np.bincount(b, minlength=nbins), out=starts[1:])
    return glo, inv, nb, starts, o[order]


def closest_point_on_triangle(p, tri):
    """Closest point on the closed triangle and its distance to p
    (broadphase.py:291-300; Ericson RTCD 5.1.5, the branch order of
    _kernels.py:159-194 and of the device closest_on_tri)."""
    tri = np.asarray(tri, dtype=np.float64).reshape(3, 3)
    area = 0.5 * np.linalg.norm(np.cross(tri[1] - tri[0], tri[2] - tri[0]))
    if area <= 0.0:
        raise ValidationError("degenerate triangle")
    p = np.asarray(p, dtype=np.float64).reshape(3)
    a, b, c = tri
    ab, ac, ap = b - a, c - a, p - a
    d1, d2 = float(ab @ ap), float(ac @ ap)
    if d1 <= 0.0 and d2 <= 0.0:
        q = a
    else:
        bp = p - b
        d3, d4 = float(ab @ bp), float(ac @ bp)
        vc = d1 * d4 - d3 * d2
        cp = p - c
        d5, d6 = float(ab @ cp), float(ac @ cp)
        vb = d5 * d2 - d1 * d6
        va = d3 * d6 - d5 * d4
        if d3 >= 0.0 and d4 <= d3:
            q = b
        elif vc <= 0.0 and d1 >= 0.0 and d3 <= 0.0:
            q = a + (d1 / (d1 - d3)) * ab
        elif d6 >= 0.0 and d5 <= d6:
            q = c
        elif vb <= 0.0 and d2 >= 0.0 and d6 <= 0.0:
            q = a + (d2 / (d2 - d6)) * ac
        elif va <= 0.0 and (d4 - d3) >= 0.0 and (d5 - d6) >= 0.0:
            q = b + ((d4 - d3) / ((d4 - d3) + (d5 - d6))) * (c - b)
        else:
            denom = 1.0 / (va + vb + vc)
            q = a + ab * (vb * denom) + ac * (vc * denom)
    return np.array(q, dtype=np.float64), float(np.linalg.norm(p - q))
