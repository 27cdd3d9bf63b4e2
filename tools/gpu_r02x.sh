mkdir -p gpurun_out
timeout 900 python tools/ab_time.py 3 40 libntbc_epi0.so libntbc.so > gpurun_out/r02x_ab.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02x_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02x_tests.log
