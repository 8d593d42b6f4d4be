# Round-end evidence refresh (run under gpurun): tests, smoke, bench lines of
# c1-c5 and the reference arm, the ncu launch list of the bench command, one
# ncu --set full capture of a c2 evaluation (summarised on the box: the
# .ncu-rep files stay in /tmp, gpurun_out is capped at 64 MiB).
set -x
OUT=${OUT:-gpurun_out/refresh}
mkdir -p $OUT /tmp/reps
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.sm --format=csv > $OUT/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> $OUT/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
for c in c2 c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_c2.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -c 40 -o /tmp/reps/full_c2 python tools/profile_one.py c2 3 > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py full /tmp/reps/full_c2.ncu-rep > $OUT/ncu_full_c2.md
python tools/ncu_summary.py launches $OUT/launches_bench_c2.csv > $OUT/launches_bench_c2.md
python tools/ncu_traffic.py /tmp/reps/full_c2.ncu-rep c2 $OUT/traffic.json
for c in c3 c4 c5; do
  timeout 900 ncu --set full --clock-control none -k regex:"k1t_gemm|k3t_gemm|k6_real" -c 3 -o /tmp/reps/full_$c python tools/profile_one.py $c 1 > $OUT/ncu_$c.log 2>&1
  python tools/ncu_traffic.py /tmp/reps/full_$c.ncu-rep $c $OUT/traffic.json
  python tools/ncu_summary.py full /tmp/reps/full_$c.ncu-rep > $OUT/ncu_full_$c.md
done
ls -la /tmp/reps
