# Evidence refresh (run under gpurun): tests, smoke, bench lines of c1-c5 and
# the reference arm, the ncu launch list of the bench command, ncu --set full
# captures (plus FP64 instruction and tensor-pipe counters) of every kernel
# of a c2 evaluation, of the GEMMs / pair kernel / binning at c3-c5 and of
# the FP64-pipe reciprocal kernels; summarised on the box (the .ncu-rep
# files stay in /tmp, gpurun_out is capped at 64 MiB).
set -x
OUT=${OUT:-gpurun_out/refresh}
mkdir -p $OUT /tmp/reps
X=$(python -c "import sys; sys.path.insert(0,'tools'); import ncu_summary; print(ncu_summary.EXTRA_METRICS)")
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.sm --format=csv > $OUT/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> $OUT/gpu.txt
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
fi
for c in c2 c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_c2.json 2> $OUT/bench_ref.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > $OUT/plain_l.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > $OUT/ncu_l.log 2>&1
python tools/ncu_summary.py launches $OUT/launches_bench_c2.csv > $OUT/launches_bench_c2.md
python tools/profile_one.py c2 3 > $OUT/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --metrics $X --clock-control none --import-source on -c 40 -o /tmp/reps/full_c2 python tools/profile_one.py c2 3 > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py full /tmp/reps/full_c2.ncu-rep > $OUT/ncu_full_c2.md
python tools/ncu_traffic.py /tmp/reps/full_c2.ncu-rep c2 $OUT/traffic.json
python tools/ncu_lines.py /tmp/reps/full_c2.ncu-rep rs_pairs 40 > $OUT/ncu_lines_c2_k6.txt
for c in c3 c4 c5; do
  python tools/profile_one.py $c 1 > $OUT/plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --metrics $X --clock-control none -k regex:"k1t_gemm|k3t_gemm|k6_real|k4_bin|k5_|k_unpermute|k2p_final" -c 10 -o /tmp/reps/full_$c python tools/profile_one.py $c 1 > $OUT/ncu_$c.log 2>&1
  python tools/ncu_traffic.py /tmp/reps/full_$c.ncu-rep $c $OUT/traffic.json
  python tools/ncu_summary.py full /tmp/reps/full_$c.ncu-rep > $OUT/ncu_full_$c.md
done
# the FP64-pipe reciprocal kernels (ewb_set_tensor_cores(0)) at c2 and c5
for c in c2 c5; do
  python tools/profile_one.py $c 1 fp64 > $OUT/plain_fp64_$c.log 2>&1 && \
  timeout 900 ncu --set full --metrics $X --clock-control none -k regex:"k1_structure|k3_force_gather|k3c_force" -c 4 -o /tmp/reps/fp64_$c python tools/profile_one.py $c 1 fp64 > $OUT/ncu_fp64_$c.log 2>&1
  python tools/ncu_summary.py full /tmp/reps/fp64_$c.ncu-rep > $OUT/ncu_fp64_$c.md
  python tools/ncu_traffic.py /tmp/reps/fp64_$c.ncu-rep ${c}_fp64 $OUT/traffic.json
done
ls -la /tmp/reps
