mkdir -p gpurun_out
timeout 900 python tools/ab_time.py 3 40 libntbc.so libntbc_pp.so > gpurun_out/r02j_ab.log 2>&1
NTBC_LIB=libntbc_pp.so timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c1_full or c2_full or 4k_sampled or ragged or conservative or extreme or full_material_digests or naive or odd_coarsest or mirror" > gpurun_out/r02j_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02j_tests.log
