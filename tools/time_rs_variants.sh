#!/bin/bash
# real-space stage time (tools/rs_time.py) of every variants/lib_*.so
for so in variants/lib_*.so; do
  echo "== $so"
  EWALDB200_LIB=$PWD/$so timeout 300 python tools/rs_time.py "$@" 2>&1 | tail -n 4
done
