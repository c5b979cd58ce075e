#!/bin/bash
# round-2 GPU check: sanitizer runs + ncu captures of the current hot kernels
set -u
O=gpurun_out/r2
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
for tool in memcheck racecheck synccheck; do
  for tgt in mine select; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_targets.py $tgt > $O/san_${tool}_${tgt}.log 2>&1; echo "$tool $tgt rc=$?" >> $O/san_summary.txt
  done
  for mode in two-pass ticket pipe; do
    SAN_SESSIONS=20000 SAN_STEPS=3 PASTE_LIVE_MODE=$mode timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_targets.py live > $O/san_${tool}_live_${mode}.log 2>&1; echo "$tool live $mode rc=$?" >> $O/san_summary.txt
  done
done
timeout 300 $NCU -k regex:'predict_live_kernel' -s 3 -c 1 -o $O/ncu_live python scripts/ncu_predict.py > $O/ncu_live.log 2>&1
timeout 300 $NCU -k regex:'predict_live_stage|live_scatter' -s 2 -c 2 -o $O/ncu_serve python scripts/ncu_predict.py > $O/ncu_serve.log 2>&1
timeout 300 $NCU -k regex:'leaf_' -c 3 -o $O/ncu_leaf python scripts/ncu_leaf.py > $O/ncu_leaf.log 2>&1
timeout 300 $NCU -k regex:'replay|predict' -s 2 -c 3 -o $O/ncu_replay python scripts/profile_replay.py > $O/ncu_replay.log 2>&1
for r in live serve leaf replay; do python profiles/summarize_ncu.py $O/ncu_$r.ncu-rep ncu_${r}_r2 > $O/ncu_${r}_r2.json 2>>$O/summ.err; done
cat $O/san_summary.txt
