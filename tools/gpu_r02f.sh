mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "pack" tests/test_gpu_checked.py -q -p no:cacheprovider > gpurun_out/r02f_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02f_tests.log
for i in 1 2; do
NTBC_LIB=libntbc.so python tools/pack_bench.py r02f_pal2 20 > gpurun_out/r02f_pack_pal2_$i.log 2>&1
NTBC_LIB=libntbc_pal0.so python tools/pack_bench.py r02f_pal0 20 > gpurun_out/r02f_pack_pal0_$i.log 2>&1
done
cp profiles/pack_r02f_pal2.json profiles/pack_r02f_pal0.json gpurun_out/ 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -c 1 -o gpurun_out/r02f_pack \
  python tools/pack_bench.py r02f_ncu 2 > gpurun_out/r02f_ncu_pack.log 2>&1
