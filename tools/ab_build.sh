#!/bin/bash
# A/B helper: rebuild the library with extra nvcc flags and run a short bench line.
# usage: tools/ab_build.sh "<nvcc extra flags>" [bench args...]
set -e
export KVMIX_NVCC_EXTRA="$1"; shift
python -c "import __graft_entry__ as g; g.build(force=True)" 2>&1 | grep -iE "error" || true
timeout 150 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$KVMIX_NVCC_EXTRA', '$*', round(d['value'],1), round(d['roofline']['achieved'],1), round(d['roofline']['frac'],4))"
