#!/bin/bash
# S26-only timing: classes over 64 roots + 4 roots' layers.  usage: tools/quick2.sh <tag>
tag=${1:-x}
python tools/diag.py --scale 26 --roots 64 --quiet --classes > gpurun_out/classes_s26_$tag.log 2>&1
tail -7 gpurun_out/classes_s26_$tag.log
python tools/diag.py --scale 26 --roots 4 > gpurun_out/layers_s26_$tag.log 2>&1
grep root gpurun_out/layers_s26_$tag.log
