#!/bin/bash
# DBG=1 build, then the switch sweep of scripts/gpu_dbg.sh on one layer; rebuilds the normal library after.
OUT=gpurun_out/${1:-dbg2}
shift
mkdir -p $OUT
touch paper_2410_23745_b200/csrc/tc.cu && make DBG=1 -j8 > $OUT/build.log 2>&1
bash scripts/gpu_dbg.sh $(basename $OUT) "$@"
touch paper_2410_23745_b200/csrc/tc.cu && make -j8 > /dev/null 2>&1
