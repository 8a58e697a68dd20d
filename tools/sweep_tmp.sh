python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/sweep.txt
for f in paper_2508_16121_b200/_lib/variants/lib*.so; do
  echo "== $f" >> gpurun_out/sweep.txt
  SVDLUT_LIB=$f timeout 120 python tools/kbench.py --variant 0 --reps 100 $SWEEP_ARGS >> gpurun_out/sweep.txt 2>&1
done
