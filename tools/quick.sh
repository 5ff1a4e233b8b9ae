#!/bin/bash
# Quick GPU check of a kernel change: parity subset, then per-class timings at
# SCALE 26 / SCALE 20 / uniform 2^22 (tools/diag.py).  usage: tools/quick.sh <tag>
tag=${1:-x}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_mgpu.py tests/test_layers.py -m gpu -x -q > gpurun_out/t_$tag.log 2>&1
tail -3 gpurun_out/t_$tag.log
python tools/diag.py --scale 26 --roots 64 --quiet --classes > gpurun_out/classes_s26_$tag.log 2>&1
tail -7 gpurun_out/classes_s26_$tag.log
python tools/diag.py --scale 26 --roots 4 > gpurun_out/layers_s26_$tag.log 2>&1
grep root gpurun_out/layers_s26_$tag.log
python tools/diag.py --scale 20 --roots 64 --quiet --classes 2>&1 | tail -6
python tools/diag.py --scale 22 --uniform --roots 64 --quiet --classes 2>&1 | tail -5
