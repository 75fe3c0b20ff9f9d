#!/bin/bash
# Bounds-checked debug build (-DMPMB_DEVICE_CHECKS=1: every hot-path slot / node / shared-memory
# index checked, a violation traps with its site) run over the sanitizer workload and the GPU
# parity tests; the substitute for compute-sanitizer, which the GPU pool does not allow.
set -u
mkdir -p gpurun_out
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so
# built in this container: make -C paper_2502_18437_b200 BUILD=build_checks LIB=libmpm_b200_checks.so NVFLAGS_EXTRA=-DMPMB_DEVICE_CHECKS=1
cp paper_2502_18437_b200/libmpm_b200_checks.so paper_2502_18437_b200/libmpm_b200.so
python tools/sanitize_run.py > gpurun_out/device_checks.txt 2>&1; echo "workload rc=$?" | tee -a gpurun_out/device_checks.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dd.py tests/test_gpu_scale.py tests/test_gpu_results.py -m gpu -q -x >> gpurun_out/device_checks.txt 2>&1
echo "tests rc=$?" | tee -a gpurun_out/device_checks.txt
grep -c "MPMB_DCHECK failed" gpurun_out/device_checks.txt
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so
