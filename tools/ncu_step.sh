#!/bin/bash
# ncu --set full over one pipelined engine step (tools/launch_list.py); exports the raw page as
# CSV on the box and drops the (large) report so gpurun_out/ stays under the copy-back limit.
#   bash tools/ncu_step.sh <tag> [extra env...]
tag=${1:-step}
out=gpurun_out/${tag}
ncu --set full --import-source on --clock-control none --profile-from-start off -o ${out} \
    python tools/launch_list.py > ${out}.log 2>&1
echo "ncu rc=$?"
ncu -i ${out}.ncu-rep --page raw --csv > ${out}_raw.csv 2>> ${out}.log
echo "export rc=$? $(wc -c < ${out}_raw.csv) bytes"
gzip -f ${out}_raw.csv
rm -f ${out}.ncu-rep
