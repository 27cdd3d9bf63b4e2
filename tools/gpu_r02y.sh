mkdir -p gpurun_out
timeout 900 python tools/ab_time.py 3 40 libntbc.so libntbc_epi2.so libntbc_epi0.so > gpurun_out/r02y_ab.log 2>&1
NTBC_LIB=libntbc_epi2.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider -k "c1_full or c2_full or 4k_sampled or ragged or extreme or full_material_digests or odd_coarsest or mirror or conservative or fuzz" > gpurun_out/r02y_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02y_tests.log
