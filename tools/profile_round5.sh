# Fifth profiling pass of the round (run under gpurun): bench lines for every
# config, launch list of the headline, full ncu of forward and backward.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_r01g.json 2> gpurun_out/bench_r01g.err
for c in 3 4 5; do timeout 600 python bench.py --config $c 2>/dev/null | tail -1 >> gpurun_out/bench_configs_r01g.jsonl; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r01g.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e \
  > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_fwd_kernel -s 4 -c 1 \
  -o gpurun_out/fwd_r01g python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/fwd_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_bwd_kernel -c 1 \
  -o gpurun_out/bwd_r01g python bench.py --config 5 --steps 1 --warmup 1 --no-graph > gpurun_out/bwd_full.log 2>&1
timeout 300 python tools/runtime_table.py --out gpurun_out/runtime_table_r01g.txt > /dev/null 2>&1
ls -la gpurun_out
