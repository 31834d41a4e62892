#!/bin/bash
# Memory-safety evidence without compute-sanitizer (closed on this pool): the bounds-checked
# build, three poison bytes for the library scratch, canaries after caller buffers, oracle
# checks; the three runs' result digests must be identical.  Output: gpurun_out/sanitize_*.log
set -u
mkdir -p gpurun_out
LIB=build/checked/libpaircount.so
test -f $LIB || { echo "missing $LIB (python -m paper_1901_11204_b200.build --checked)"; exit 1; }
rc=0
for p in 0x00 0xA5 0xFF; do
  PAIRCOUNT_LIB=$LIB PAIRCOUNT_POISON=$p timeout 900 python scripts/sanitize_cases.py > gpurun_out/sanitize_$p.log 2>&1
  r=$?; echo "poison $p rc=$r"; [ $r -ne 0 ] && rc=1 && tail -20 gpurun_out/sanitize_$p.log
done
grep -h "^DIGEST" gpurun_out/sanitize_0x*.log | sort | uniq -c | awk '{print "digest variants:", NR, "count", $1}'
n=$(grep -h "^DIGEST" gpurun_out/sanitize_0x*.log | sort -u | wc -l)
[ "$n" = "1" ] && echo "DIGESTS IDENTICAL across poison bytes" || { echo "DIGESTS DIFFER ($n variants)"; rc=1; }
exit $rc
