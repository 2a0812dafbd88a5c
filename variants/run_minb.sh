#!/bin/bash
bash variants/ab.sh base MINB_FWD10 MINB_FWD12 MINB_FWD_ALPHA10 MINB_BWD7 base > gpurun_out/ab_minb.txt 2>&1
cat gpurun_out/ab_minb.txt
