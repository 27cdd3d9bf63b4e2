mkdir -p gpurun_out
for i in 1 2; do
NTBC_LIB=libntbc_prev.so python tools/pack_bench.py r02i_prev 20 > gpurun_out/r02i_pack_prev_$i.log 2>&1
NTBC_LIB=libntbc.so python tools/pack_bench.py r02i_new 20 > gpurun_out/r02i_pack_new_$i.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -k "pack" tests/test_gpu_checked.py -q -p no:cacheprovider > gpurun_out/r02i_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02i_tests.log
timeout 900 python -m pytest tests/test_gpu_checked.py -q -p no:cacheprovider >> gpurun_out/r02i_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02i_tests.log
