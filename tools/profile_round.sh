# Round profiling pass (run under gpurun): bench lines (configs 1-5, reference
# arm), launch list, full ncu of the forward and backward kernels, the
# shared-memory / texture / atomic microbenchmarks and the runtime table.
# Outputs in gpurun_out/ (summarised into profiles/ by tools/ncu_summary.py).
set -x
R=${1:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
for c in 1 3 4 5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 >> gpurun_out/bench_configs_$R.jsonl 2>> gpurun_out/bench_configs_$R.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_$R.json 2> gpurun_out/bench_reference_$R.err
timeout 600 python bench.py --impl reference --config 1 --steps 3 >> gpurun_out/bench_reference_$R.json 2>> gpurun_out/bench_reference_$R.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra \
  > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_fwd_kernel -s 4 -c 1 \
  -o gpurun_out/fwd_$R -f python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > gpurun_out/fwd_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_bwd_kernel -c 1 \
  -o gpurun_out/bwd_$R -f python tools/bwd_once.py > gpurun_out/bwd_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_bwd_kernel -s 1 -c 1 \
  -o gpurun_out/l2step_$R -f python tools/bwd_once.py > gpurun_out/l2step_ncu.log 2>&1
for m in ldsclean texphase atomswidth atomspat shfllds; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/$m tools/microbench/$m.cu
done
{ ./tools/microbench/ldsclean tools/microbench/clean.txt; ./tools/microbench/ldsclean tools/microbench/clean2.txt;
  ./tools/microbench/texphase; ./tools/microbench/atomswidth; ./tools/microbench/atomspat tools/microbench/bwd_atoms.txt;
  ./tools/microbench/ldsclean tools/microbench/bwd_lds.txt; ./tools/microbench/shfllds; } > gpurun_out/microbench_$R.txt 2>&1
timeout 600 python tools/runtime_table.py > gpurun_out/runtime_table_$R.txt 2>&1
ls -la gpurun_out
