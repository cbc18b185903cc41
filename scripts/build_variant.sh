#!/bin/bash
# Variant builds of the library for A/B timing (scripts/ab_time.py with HD_LIBRARY):
#   scripts/build_variant.sh NAME -DFLAG=VALUE ...   ->  _ab/libhelmdef_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p _ab
python -c "from paper_2010_10232_b200 import build as b; b.build()" >/dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I include -lineinfo "$@" \
  -c paper_2010_10232_b200/csrc/solver.cu -o _ab/solver_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC _ab/solver_$name.o \
  paper_2010_10232_b200/_build/assembly.cpp.o paper_2010_10232_b200/_build/banded.cpp.o \
  -o _ab/libhelmdef_$name.so -lcublas -lcusolver -lcudart -ldl
echo _ab/libhelmdef_$name.so
