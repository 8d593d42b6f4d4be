#!/bin/bash
# whole-evaluation time (tools/overlap_ab.py: sequential vs two streams) of every variants/lib_*.so
for so in variants/lib_*.so; do
  echo "== $so"
  EWALDB200_LIB=$PWD/$so timeout 300 python tools/overlap_ab.py "$@" 2>&1 | grep "overlap=True"
done
