set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/t_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/t_gpu_tests.log
timeout 600 python bench.py > gpurun_out/t_bench.json 2> gpurun_out/t_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/t_bench_ref.json 2> gpurun_out/t_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/t_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/t_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_decode -c 1 -o gpurun_out/r01t python tools/profile_step.py 3 2 > gpurun_out/t_ncu_full.log 2>&1
ls -la gpurun_out
