#!/bin/bash
mkdir -p gpurun_out
python scripts/debug_big.py > gpurun_out/debug_big_new.log 2>&1
GP_LIB=paper_2410_12707_b200/_lib/variants/old/libadatopk.so python scripts/debug_big.py > gpurun_out/debug_big_old.log 2>&1
cat gpurun_out/debug_big_new.log gpurun_out/debug_big_old.log
