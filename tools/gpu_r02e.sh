mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_checked.py "tests/test_gpu_parity.py::test_full_material_digests" -q -s -p no:cacheprovider > gpurun_out/r02e_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02e_tests.log
