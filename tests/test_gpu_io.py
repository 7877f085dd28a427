"""Frame output from device snapshots (io.py:120-196):
write_sphere_csv assembles its columns on the device (gf_sphere_frame) and
must produce the reference's text for the same state byte for byte; here
the expected text is built from the oracle's restatement of the reference's
sphere-world transform on the downloaded state."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_04648_b200 import io as gio
from paper_2311_04648_b200 import scenes

pytestmark = pytest.mark.gpu


def _fmt(x):
    return format(float(x), ".17g")


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_sphere_csv_byte_identical(tmp_path, precision):
    sim = scenes.settling_box(2_000, precision=precision)
    sim.initialize()
    with sim:
        sim.do_dynamics(50 * sim.h)
        path = tmp_path / "frame.csv"
        gio.write_sphere_csv(sim, path, content=("XYZ", "ABSV", "FAMILY", "VEL"))
        sim._sync_all()
        s = sim.store
        n = s.n_owners
        pos = O.decode_positions(s.voxel[:n], s.subvoxel[:n], s.domain.lo, float(s.domain.voxel_edge))
        sph = sim._sph_geom
        centres, _ = O.sphere_world(sph, s.geom_params[:s.n_geoms], s.geom_owner[:s.n_geoms], pos, s.quat[:n])
        owners = s.geom_owner[sph]
        vel = s.lin_vel[owners].astype(np.float64)
        absv = np.sqrt((vel ** 2).sum(axis=1))
        fam = s.owner_family[owners]
        lines = ["x,y,z,absv,family,vx,vy,vz"]
        for k in range(sph.shape[0]):
            lines.append(",".join([_fmt(centres[k, 0]), _fmt(centres[k, 1]), _fmt(centres[k, 2]), _fmt(absv[k]),
                                   str(int(fam[k])), _fmt(vel[k, 0]), _fmt(vel[k, 1]), _fmt(vel[k, 2])]))
        assert path.read_text() == "\n".join(lines) + "\n"


def test_mesh_vtk_frame(tmp_path):
    sim = scenes.rover_wheel(6_000, packing="lattice", precision="f64", h=2e-6, v_err=3.0, n_max=4, sinkage=0.0005,
                             wheel_radius=0.05, aspect=2.0)
    sim.initialize()
    with sim:
        sim.do_dynamics(20 * sim.h)
        path = tmp_path / "wheel.vtk"
        gio.write_mesh_vtk(sim, path)
        text = path.read_text().split("\n")
        n_tri = int(np.sum(sim.store.geom_kind[:sim.store.n_geoms] == 1))
        assert text[4] == f"POINTS {3 * n_tri} double"
        assert f"CELLS {n_tri} {4 * n_tri}" in text
