#!/bin/bash
# A/B of two librsk builds on one GPU box, back to back (base = the in-tree build, var =
# the build at $2): per-phase probe of the streaming loop at 1 / 4 / 16 / 32 active shifts,
# twice each, interleaved.   usage: bash tools/ab_probe.sh <tag> <path/to/variant/librsk.so>
out=gpurun_out/ab_$1
mkdir -p $out
for m in 1 4 16 32; do
  for v in base var base var; do
    if [ $v = base ]; then lp=""; else lp="RSK_LIB_PATH=$2"; fi
    env $lp timeout 300 python tools/probe_defl.py C4 $m 40 >> $out/probe_${v}_m$m.log 2>&1
  done
done
