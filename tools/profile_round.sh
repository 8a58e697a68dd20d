# Round profiling pass (run under gpurun): bench line, launch list, full ncu of
# the forward and backward kernels.  Outputs in gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e \
  > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_fwd_kernel -s 4 -c 1 \
  -o gpurun_out/fwd_full python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/fwd_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_bwd_kernel -c 1 \
  -o gpurun_out/bwd_full python bench.py --config 5 --steps 1 --warmup 1 --no-graph > gpurun_out/bwd_full.log 2>&1
ls -la gpurun_out
