#!/bin/bash
# Diagnostic build: libcachetune_b200 with the attention timeline trace
# (CT_ATT_TRACE) -> tools/probes/bin/lib_trace.so.  Not the product library.
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2605_24022_b200 import _build; _build.build()"
mkdir -p build/trace tools/probes/bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Iinclude -DCT_ATT_TRACE -c paper_2605_24022_b200/csrc/attention_tc.cu \
  -o build/trace/attention_tc.o
objs=$(ls build/obj/*.o | grep -v attention_tc.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/probes/bin/lib_trace.so \
  build/trace/attention_tc.o $objs -lcudart_static -ldl -lrt -lpthread
echo built tools/probes/bin/lib_trace.so
