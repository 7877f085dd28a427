#!/bin/bash
# Stage (in this container, where /root/reference exists) or run (on the GPU
# box) the reference's own tests through the drop-in.
#   tools/reftests/run.sh stage   copy pkg/tests/test_{core,broadphase,forces,engine}.py
#                                 into baseline/reftests/ (git-ignored)
#   tools/reftests/run.sh run     pytest them; the pass list goes to gpurun_out/reftests.txt
set -e
cd "$(dirname "$0")/../.."
D=baseline/reftests
if [ "$1" = stage ]; then
  mkdir -p $D
  for t in test_core test_broadphase test_forces test_engine; do cp /root/reference/pkg/tests/$t.py $D/; done
  cp tools/reftests/conftest.py $D/conftest.py
  exit 0
fi
mkdir -p gpurun_out
timeout 1500 python -m pytest $D -q -p no:cacheprovider -rA -m "not slow" > gpurun_out/reftests.txt 2>&1 || true
tail -5 gpurun_out/reftests.txt
