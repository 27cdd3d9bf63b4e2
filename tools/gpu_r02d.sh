mkdir -p gpurun_out
./tools/micro/selu_rate > gpurun_out/r02d_selu_rate.txt 2>&1
timeout 900 python tools/ab_time.py 3 40 libntbc.so libntbc_mufu.so libntbc_nogrid.so > gpurun_out/r02d_ab.log 2>&1
NTBC_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 2 --steps 3 --warmup 3 --materials 4 --no-cpu-baseline > gpurun_out/r02d_bench_n2_onegpu.json 2> gpurun_out/r02d_bench_n2_onegpu.err
echo "exit $?" >> gpurun_out/r02d_bench_n2_onegpu.err
