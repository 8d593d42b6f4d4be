#!/bin/bash
# time every variants/lib_*.so on the given configs
for so in variants/lib_*.so; do
  echo "== $so"
  EWALDB200_LIB=$PWD/$so timeout 300 python tools/quick_time.py "$@" 2>&1 | grep -v "^c. {" | awk "NR%4==0"
done
