"""Runs the REFERENCE's own tests (grainforge pkg/tests) against this
package: `grainforge` and its submodules are aliased to
paper_2311_04648_b200 before the test modules import them.

tools/reftests/run.sh copies the reference's test files next to this
conftest under baseline/reftests/ (git-ignored: the reference's sources are
not part of this repo) and runs them on the GPU box."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2311_04648_b200 as pkg  # noqa: E402
from paper_2311_04648_b200 import broadphase, core, engine, forces, types  # noqa: E402

sys.modules["grainforge"] = pkg
for name, mod in (("core", core), ("broadphase", broadphase), ("forces", forces), ("engine", engine),
                  ("types", types)):
    sys.modules[f"grainforge.{name}"] = mod
    setattr(pkg, name, mod)
