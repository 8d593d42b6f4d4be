set -x
mkdir -p gpurun_out/r01f
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.sm --format=csv > gpurun_out/r01f/gpu.txt
for c in c2 c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r01f/bench_$c.json 2> gpurun_out/r01f/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01f/bench_ref_c2.json 2> gpurun_out/r01f/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01f/launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01f/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -c 40 -o gpurun_out/r01f/full_c2 python tools/profile_one.py c2 3 > gpurun_out/r01f/ncu_full.log 2>&1
