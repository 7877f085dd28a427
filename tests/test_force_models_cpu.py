"""User force models: NVRTC compile checks (CPU, no device) and the plugin
registry semantics (forces.py:360-440)."""

import pytest

import paper_2311_04648_b200 as gf
from paper_2311_04648_b200 import forces, models


def test_cohesive_model_compiles_with_nvrtc():
    m = models.cohesive_model()
    assert m.cuda_src and m.pair_props[-1] == "coh"
    forces.compile_check(m)  # raises on any NVRTC error


def test_broken_source_reports_compiler_error():
    bad = gf.ForceModel(name="broken_model_for_test", wildcards=("w",), pair_props=(),
                        device_kernel="nvrtc", cuda_src="__device__ void user_core(int x) { y = 1; }")
    with pytest.raises(gf.ConfigurationError, match="does not compile"):
        forces.compile_check(bad)


def test_registry():
    assert gf.get_force_model("hertz_mindlin") is forces.DEFAULT_MODEL
    with pytest.raises(gf.ConfigurationError):
        gf.get_force_model("nope")
    with pytest.raises(gf.ConfigurationError, match="already registered"):
        gf.register_force_model(forces.DEFAULT_MODEL)
    with pytest.raises(gf.ConfigurationError, match="no compiled device kernel"):
        gf.register_force_model(gf.ForceModel(name="x", wildcards=(), pair_props=(),
                                              device_kernel="something"))


def test_missing_property_named():
    mt = gf.MaterialTable()
    mt.load_material({"E": 1e8, "nu": 0.3, "CoR": 0.5, "mu": 0.3, "Crr": 0.0})
    with pytest.raises(gf.ConfigurationError, match="coh"):
        forces.material_pair_stack(mt, models.cohesive_model())
