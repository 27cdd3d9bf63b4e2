# Round-end evidence: GPU tests, smoke, bench line (+ reference arm, torchrun N=1, C5 batch at N=1), ncu launch
# list + --set full captures (fused, pack), Tab. 1, pack bench, A/B timing of C2/C3/C4.  usage: bash tools/gpu_final.sh <tag>
tag=${1:-final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
nproc > gpurun_out/${tag}_nproc.txt; lscpu | grep "Model name" >> gpurun_out/${tag}_nproc.txt
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/${tag}_gpu_tests.log
for f in faithfulness_gpu contract_f_gpu contract_p_gpu; do cp gpurun_out/$f.json gpurun_out/${tag}_$f.json 2>/dev/null; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-pack > gpurun_out/${tag}_bench_torchrun.json 2> gpurun_out/${tag}_bench_torchrun.err
timeout 900 python bench.py --materials 64 --steps 5 --warmup 3 --no-cpu-baseline --no-pack > gpurun_out/${tag}_bench_c5_n1.json 2> gpurun_out/${tag}_bench_c5_n1.err
timeout 900 python tools/ab_time.py 2 40 libntbc.so > gpurun_out/${tag}_c2.log 2>&1
timeout 900 python tools/ab_time.py 4 40 libntbc.so > gpurun_out/${tag}_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pack > gpurun_out/${tag}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_decode -c 1 -o gpurun_out/${tag} \
  python tools/profile_step.py 3 2 > gpurun_out/${tag}_ncu_full.log 2>&1
NTBC_CONTRACT=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_decode -c 1 -o gpurun_out/${tag}_p \
  python tools/profile_step.py 3 2 > gpurun_out/${tag}_ncu_full_p.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -c 1 -o gpurun_out/${tag}_pack \
  python tools/pack_bench.py ${tag} 2 > gpurun_out/${tag}_ncu_pack.log 2>&1
# summaries on the box (gpurun copies back at most 64 MiB): contract P first, then H (latest_fused_traffic.json = H)
python tools/ncu_summary.py gpurun_out/${tag}_p.ncu-rep ${tag}_p > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${tag}.ncu-rep ${tag} > /dev/null 2>&1
cp profiles/${tag}_p_fused_ncu.* profiles/${tag}_fused_ncu.* profiles/latest_fused_traffic.json gpurun_out/ 2>/dev/null
ncu -i gpurun_out/${tag}_pack.ncu-rep --page raw --csv > gpurun_out/${tag}_pack_raw.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/${tag}.ncu-rep 16777216 60 > gpurun_out/${tag}_lines.txt 2>/dev/null
mv gpurun_out/${tag}_p.ncu-rep gpurun_out/${tag}_pack.ncu-rep /tmp/ 2>/dev/null
python tools/tab1.py ${tag} 20 > gpurun_out/${tag}_tab1.log 2>&1; cp profiles/tab1_${tag}.json gpurun_out/
NTBC_CONTRACT=2 python tools/tab1.py ${tag}_p 20 > gpurun_out/${tag}_tab1_p.log 2>&1; cp profiles/tab1_${tag}_p.json gpurun_out/
python tools/pack_bench.py ${tag} 20 > gpurun_out/${tag}_pack.log 2>&1; cp profiles/pack_${tag}.json gpurun_out/
du -sh gpurun_out; ls -la gpurun_out | tail -5
