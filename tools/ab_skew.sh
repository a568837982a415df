#!/bin/bash
# A/B of the lockstep and the skewed (RSK_STREAM_SKEW=1) schedule of the streaming loop on
# one box, interleaved: two groups (halves = groups) and one group (halves split it).
# usage: bash tools/ab_skew.sh <tag>
out=gpurun_out/ab_skew_$1
mkdir -p $out
for og in 0 1; do
  for m in 1 2 4 8 16 32; do
    for v in 0 1 0 1; do
      if [ $og = 1 ]; then e="PROBE_ONE_GROUP=1"; else e="PROBE_TWO=1"; fi
      env $e RSK_STREAM_SKEW=$v timeout 300 python tools/probe_defl.py C4 $m 40 2>&1 | tail -2 >> $out/probe_og${og}_skew${v}_m$m.log
    done
  done
done
grep -H "per lockstep" $out/*.log | sed 's/.*probe_//' | awk '{print $1, $NF}'
