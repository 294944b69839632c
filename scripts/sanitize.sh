#!/bin/bash
# compute-sanitizer runs of the GPU suite's small cases (memcheck, racecheck, synccheck, initcheck).
# Writes profiles-ready logs to gpurun_out/sanitizer_<tool>.log; exit code = number of failing tools.
cd "$(dirname "$0")/.."
SEL="tests/test_gpu_parity.py::test_small_images_vs_reference_digests tests/test_gpu_parity.py::test_block_api_known_answers tests/test_gpu_robustness.py::test_large_slot_blocks_into_dirty_buffer tests/test_gpu_slide.py::test_slide_device_archive_vs_oracle tests/test_gpu_region.py tests/test_gpu_parity.py::test_corrupted_containers_same_error_class"
SEL2="tests/test_gpu_parity.py::test_small_images_vs_reference_digests tests/test_gpu_parity.py::test_block_api_known_answers tests/test_gpu_robustness.py::test_large_slot_blocks_into_dirty_buffer tests/test_gpu_slide.py::test_slide_device_archive_vs_oracle"
fails=0
for tool in memcheck racecheck synccheck; do
  sel="$SEL"; [ $tool != memcheck ] && sel="$SEL2"
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
    --log-file gpurun_out/sanitizer_${tool}.log python -m pytest $sel -x -q -p no:cacheprovider \
    > gpurun_out/sanitizer_${tool}.pytest.log 2>&1
  rc=$?
  echo "$tool rc=$rc" | tee -a gpurun_out/sanitizer_summary.txt
  tail -3 gpurun_out/sanitizer_${tool}.pytest.log >> gpurun_out/sanitizer_summary.txt
  tail -3 gpurun_out/sanitizer_${tool}.log >> gpurun_out/sanitizer_summary.txt
  [ $rc -ne 0 ] && fails=$((fails+1))
done
exit $fails
