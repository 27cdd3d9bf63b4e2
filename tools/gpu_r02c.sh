mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/r02c_gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02c_gpu_tests.log
timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
python tools/tab1.py r02c 20 > gpurun_out/r02c_tab1.log 2>&1
NTBC_PAIR_LAUNCHES=1 python tools/tab1.py r02c_2l 20 > gpurun_out/r02c_tab1_2launch.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_target.py 1 > gpurun_out/r02c_memcheck_c1.log 2>&1; echo "exit $?" >> gpurun_out/r02c_memcheck_c1.log
