#!/bin/bash
# compute-sanitizer over every kernel path (tests/sanitize_run.py: small seeded problems plus the
# configs[1] rollout problem, each checked against the oracle).  Logs to gpurun_out/<tag>_<tool>.log.
#   gpurun -- 'bash bench/sanitize.sh r02'
tag=${1:-r02}
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
$CS --version > gpurun_out/${tag}_sanitizer_version.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 700 $CS --tool $tool $extra --target-processes all --print-limit 100 \
      python tests/sanitize_run.py > gpurun_out/${tag}_sanitize_${tool}.log 2>&1
  echo "$tool exit $?" >> gpurun_out/${tag}_sanitize_summary.txt
  tail -3 gpurun_out/${tag}_sanitize_${tool}.log >> gpurun_out/${tag}_sanitize_summary.txt
done
