#!/bin/bash
# MLP GEMM variant comparison (experiment helper; not part of the product)
for v in "$@"; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; unset WIPES_GEMM_SIMPLE; elif [ "$v" = "simple" ]; then unset WIPES_LIB; export WIPES_GEMM_SIMPLE=1; else unset WIPES_GEMM_SIMPLE; export WIPES_LIB=$PWD/variants/$v.so; fi
  echo "$v $(timeout 120 python tools/bench_mlp.py 300000 1)"
done
