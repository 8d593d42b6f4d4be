# component timings of the tensor-core stages (sequential stages): 0 full,
# 1 no operand production, 2 no MMAs, 3 neither (copies, prep, epilogue).
# Each mode is a separate build (-DEWB_TC_DBG=d); the product library never
# reads it.
for d in 0 1 2 3; do
  so=/tmp/libewaldb200_dbg$d.so
  nvcc -gencode=arch=compute_100a,code=sm_100a -O3 -std=c++17 -DEWB_TC_DBG=$d -I include \
       -Xcompiler -fPIC -shared -o $so paper_1708_01135_b200/csrc/ewald_b200.cu
  echo "dbg=$d"; EWALDB200_LIB=$so python tools/rs_time.py ${@:-c2 c3 c5} 2>&1 | grep alg
done
