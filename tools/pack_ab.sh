# GPU-box helper: pack kernel variants (parity + timing), then one ncu --set full capture of pack_kernel.
# usage (via gpurun): bash tools/pack_ab.sh <tag> lib.so [lib.so ...]
tag=$1; shift
mkdir -p gpurun_out
for L in "$@"; do
  echo "== $L" >> gpurun_out/packab.log
  NTBC_LIB=$L timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pack" >> gpurun_out/packab.log 2>&1
  NTBC_LIB=$L timeout 300 python tools/pack_bench.py ab 30 >> gpurun_out/packab.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 2 -c 1 -o gpurun_out/${tag}_pack \
  python tools/pack_bench.py ab 3 > gpurun_out/${tag}_pack_ncu.log 2>&1
