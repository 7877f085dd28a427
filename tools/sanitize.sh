#!/bin/bash
# compute-sanitizer over representative GPU tests (memcheck, racecheck,
# synccheck, initcheck); summaries to gpurun_out/sanitizer_<tool>.txt
mkdir -p gpurun_out
T="tests/test_gpu_parity.py::test_dt_step_f32_within_tolerance tests/test_gpu_parity.py::test_dt_step_f64_bit_exact tests/test_gpu_parity.py::test_async_schedule_matches_oracle_stepper tests/test_gpu_parity.py::test_detect_polydisperse_with_big_spheres_vs_oracle tests/test_gpu_ref_abi.py tests/test_gpu_engine.py::test_free_fall"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
    python -m pytest $T -q -p no:cacheprovider -x > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.txt
done
