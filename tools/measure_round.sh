#!/bin/bash
# The round's committed measurements (run on one B200 through gpurun; outputs land in gpurun_out/,
# then tools/summarize_ncu.py and a copy step write profiles/):
#   smoke, the default bench line, the reference arm, the light ncu launch list, one ncu --set full
#   capture of K2 and of the K1 pair, the cfg4 head-shard lines, cfg5 at batch 64, the survey-mix line.
set -x
python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --profile-only > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_mma_kernel -s 20 -c 1 -o gpurun_out/k2_final -f python bench.py --profile-only > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"prefill_pages|int4_tokens" --launch-skip 6 -c 2 -o gpurun_out/k1_final -f python tools/k1_probe.py > /dev/null 2>&1
rm -f gpurun_out/heads.jsonl
for s in 2 4 8; do timeout 600 python bench.py --mode heads --shards $s --steps 10 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/heads.jsonl; done
timeout 900 python bench.py --batch 64 --steps 5 --warmup 3 --no-cpu-baseline --no-churn --no-k1 2>/dev/null | tail -1 > gpurun_out/cfg5_b64.json
timeout 600 python bench.py --int2-frac 0.773 --steps 10 --warmup 3 --no-cpu-baseline --no-churn --no-k1 --no-e2e 2>/dev/null | tail -1 > gpurun_out/mix773.json
# compute-sanitizer over a drive of every product kernel
python tools/sanitize_drive.py > gpurun_out/san_plain.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/san_$t.txt 2>&1
  echo "$t rc=$?"
done
