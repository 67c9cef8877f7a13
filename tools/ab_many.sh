#!/bin/bash
# A/B timing of several build_ab variants: tools/ab_many.sh script.py v1 v2 ...
# prints one JSON line per variant (SALF_LIB=build_ab/<v>/libsalf_b200.so).
S=$1; shift
for v in "$@"; do SALF_LIB=build_ab/$v/libsalf_b200.so python $S init $v 2>&1 | tail -1 | cut -c1-4000; done
