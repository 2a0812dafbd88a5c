#!/bin/bash
python tools/visible_c3.py 2>&1 | tail -2
bash variants/ab_sort.sh base rts4k base rts4k 2>&1 | grep c3
