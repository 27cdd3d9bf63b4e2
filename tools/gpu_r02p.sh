mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "pack" tests/test_gpu_checked.py -q -p no:cacheprovider > gpurun_out/r02p_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02p_tests.log
for i in 1 2; do
python tools/pack_bench.py r02p_bt 20 > gpurun_out/r02p_pack_bt_$i.log 2>&1
NTBC_PACK_WARP=1 python tools/pack_bench.py r02p_warp 20 > gpurun_out/r02p_pack_warp_$i.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -c 1 -o gpurun_out/r02p_pack \
  python tools/pack_bench.py r02p_ncu 2 > gpurun_out/r02p_ncu_pack.log 2>&1
