#!/bin/bash
# A/B two (or more) builds of libsmap.so on ONE GPU box, interleaved, so that
# box-to-box and thermal differences cancel.  On the dev box:
#   mkdir -p abtmp && cp paper_1610_07394_b200/libsmap.so abtmp/base.so
#   (edit, rebuild) && cp paper_1610_07394_b200/libsmap.so abtmp/exp.so
#   (restore the source, rebuild)
#   gpurun -- 'bash scripts/ab_libs.sh "python scripts/one.py --m 3 --n 1024 --payload atm --param 0.01 --rho 32 --gran tile --reps 12" base exp'
# then remove abtmp/.  Prints the fastest rep of each run, 3 rounds.
set -u
CMD=$1; shift
for r in 1 2 3; do
  for v in "$@"; do
    cp abtmp/$v.so paper_1610_07394_b200/libsmap.so
    echo -n "$v "; $CMD | sort -t: -k2 -n | sort -k7 -n | head -1
  done
done
