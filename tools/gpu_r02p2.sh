# contract P (binary16 selu): parity tests, checked build, A/B timing against contract H, bench sub-record
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_contract_p.py tests/test_gpu_contract_f.py tests/test_gpu_checked.py -q -s -p no:cacheprovider > gpurun_out/r02p2_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02p2_tests.log
timeout 600 python tools/ab_time.py 3 40 libntbc.so libntbc.so:NTBC_CONTRACT=2 > gpurun_out/r02p2_ab.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02p2_bench.json 2> gpurun_out/r02p2_bench.err
tail -5 gpurun_out/r02p2_tests.log; cat gpurun_out/r02p2_ab.log
