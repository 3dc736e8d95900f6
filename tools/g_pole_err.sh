#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python tools/pole_err.py > gpurun_out/pole_err.txt 2>&1
cat gpurun_out/pole_err.txt | tail -8
