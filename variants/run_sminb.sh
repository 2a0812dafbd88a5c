#!/bin/bash
bash variants/ab_sort.sh base MINB_RTS5 MINB_RTS5_MINB5 base MINB_RTS5 MINB_RTS5_MINB5 > gpurun_out/ab_sminb.txt 2>&1
cat gpurun_out/ab_sminb.txt
