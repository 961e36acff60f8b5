#!/bin/bash
# GPU test suite one file at a time, each under its own time bound (a hang stays local):
#   FILES="tests/test_gpu_x.py ..." PER_FILE=600 tests/gpu_suite.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
out=gpurun_out/r2_suite.log; : > $out
for f in ${FILES:-tests/test_gpu_*.py}; do
  timeout ${PER_FILE:-900} python -m pytest "$f" -q --tb=short -x -p no:cacheprovider > gpurun_out/r2_cur.log 2>&1
  rc=$?
  echo "== $f rc=$rc $(tail -1 gpurun_out/r2_cur.log)" >> $out
  if [ $rc -ne 0 ]; then tail -c 6000 gpurun_out/r2_cur.log >> $out; fi
done
cat $out | tail -c 12000
