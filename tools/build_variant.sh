#!/bin/bash
# Builds tools/variants/<name>.so: engine.cu recompiled with extra nvcc flags,
# linked with the in-tree setup/capi objects (dev tool for A/B kernel timing
# with tools/variant_eval.py).  Usage: tools/build_variant.sh <name> <flags...>
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p tools/variants
O=paper_2006_15367_b200/_lib/obj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" \
  -I include -I paper_2006_15367_b200/csrc -c paper_2006_15367_b200/csrc/engine.cu -o tools/variants/$name.engine.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/variants/$name.so tools/variants/$name.engine.o \
  $O/setup.cpp.o $O/setup_import.cpp.o $O/setup_gpu.cu.o $O/world.cu.o $O/capi.cu.o -Xcompiler -pthread
echo tools/variants/$name.so
