mkdir -p gpurun_out
timeout 900 python tools/ab_time.py 3 40 libntbc_prev.so libntbc.so libntbc_wpoll.so > gpurun_out/r02g_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02g_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02g_tests.log
