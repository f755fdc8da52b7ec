#!/bin/bash
# ncu full capture of one finest-level GS half-sweep launch (cfg2) for the given kernel regex
K=${1:-k_gs_stream}
OUT=${2:-gpurun_out/prof_gs_stream}
ncu --set full --import-source on --clock-control none -k "regex:$K" -s 2 -c 1 -o $OUT -f python tools/exp_gs2.py sphere
