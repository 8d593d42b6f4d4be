# component timings of the tensor-core stages (sequential stages): 0 full,
# 1 no operand production, 2 no MMAs, 3 neither (copies, prep, epilogue)
for d in 0 1 2 3; do echo "dbg=$d"; EWB_TC_DBG=$d python tools/rs_time.py ${@:-c2 c3 c5} 2>&1 | grep alg; done
