#!/bin/bash
# build libmpm_b200 variants with different compile-time knobs: NAME "FLAGS" pairs
set -e
cd "$(dirname "$0")"
make -s build/k_step.o build/k_sort.o build/k_io.o build/k_dd.o build/k_scenario.o build/k_exact.o build/engine.o build/capi.o build/dd_driver.o
mkdir -p variants
[ "${KEEP:-0}" = "1" ] || rm -f variants/*.so
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off $flags -c csrc/k_transfer.cu -o build/k_transfer_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$name.so build/k_step.o build/k_transfer_$name.o build/k_sort.o build/k_io.o build/k_dd.o build/k_scenario.o build/k_exact.o build/engine.o build/capi.o build/dd_driver.o -lcudart_static -lpthread -ldl -lrt
done
ls variants
