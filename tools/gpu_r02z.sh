mkdir -p gpurun_out
timeout 900 python tools/ab_time.py 3 40 libntbc_epi1.so libntbc.so > gpurun_out/r02z_ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_checked.py -x -q -p no:cacheprovider > gpurun_out/r02z_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02z_tests.log
