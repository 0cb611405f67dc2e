#!/bin/bash
# Bench an older package snapshot (tools/abtree/pkg_<rev>) with today's bench.py workload.
set -e
rev=$1; shift
root="$(cd "$(dirname "$0")/../.." && pwd)"
rm -rf /tmp/abold && mkdir -p /tmp/abold
cp -r "$root/tools/abtree/pkg_$rev" /tmp/abold/paper_2605_17170_b200
cp -r "$root/include" "$root/bench_data" "$root/oracle" "$root/bench.py" "$root/tools/abtree/__graft_entry__.py" /tmp/abold/
cp "$root/MEASURED_PEAKS.json" /tmp/abold/ 2>/dev/null || true
cd /tmp/abold/paper_2605_17170_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -o ../libkvmix_b200.so codec.cu decode.cu capi.cu
cd /tmp/abold
timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-k1 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rev', round(d['value'],1), round(d['roofline']['frac'],4))"
