#!/bin/bash
# compute-sanitizer over the kernels added late in round 2: the key-stream
# serving kernels (predict_live_keys_kernel, warp_scan_kernel,
# warp_copy_kernel) with the 3-byte and the 2-byte (node code) inputs, the
# scatter two-pass form for comparison, and the fused replay.
set -u
O=gpurun_out/san_r2b
mkdir -p $O
: > $O/summary.txt
for tool in memcheck racecheck synccheck; do
  for wire in 3 2; do
    W2=0; [ $wire = 2 ] && W2=1
    SAN_WIRE2=$W2 SAN_SESSIONS=20000 SAN_STEPS=4 timeout 900 compute-sanitizer --tool $tool \
      --error-exitcode 9 python scripts/sanitize_targets.py live > $O/san_${tool}_live_keys_w${wire}.log 2>&1
    echo "$tool live keys-form wire${wire}B rc=$?" >> $O/summary.txt
  done
  PASTE_LIVE_MODE=scatter SAN_SESSIONS=20000 SAN_STEPS=3 timeout 900 compute-sanitizer --tool $tool \
    --error-exitcode 9 python scripts/sanitize_targets.py live > $O/san_${tool}_live_scatter.log 2>&1
  echo "$tool live scatter rc=$?" >> $O/summary.txt
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_targets.py replay \
    > $O/san_${tool}_replay.log 2>&1
  echo "$tool replay rc=$?" >> $O/summary.txt
done
cat $O/summary.txt
