# Round capture (run under gpurun): bench lines + launch list + full ncu of the top kernel.
set -x
mkdir -p gpurun_out/cap
timeout 600 python bench.py > gpurun_out/cap/bench_c2.json 2> gpurun_out/cap/bench_c2.err
timeout 900 python bench.py --all --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cap/bench_all.json 2> gpurun_out/cap/bench_all.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/cap/bench_ref.json 2> gpurun_out/cap/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cap/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cap/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nn$ -s 1 -c 1 -o gpurun_out/cap/k_nn_c2 python tools/prof_step.py c2 2 > gpurun_out/cap/ncu_full.log 2>&1
echo done
