mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "pack" > gpurun_out/r02t_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02t_tests.log
timeout 900 python -m pytest tests/test_gpu_checked.py -q -p no:cacheprovider >> gpurun_out/r02t_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02t_tests.log
for i in 1 2; do for L in libntbc.so libntbc_bt32_2.so libntbc_bt64_1.so; do NTBC_LIB=$L python tools/pack_bench.py r02t 20 > gpurun_out/r02t_pack_${L}_$i.log 2>&1; done; done
