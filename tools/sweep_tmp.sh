python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/sweep.txt
for f in paper_2508_16121_b200/_lib/variants/lib*.so; do
  echo "== $f" >> gpurun_out/sweep.txt
  SVDLUT_LIB=$f timeout 120 python tools/kbench.py --variant 0 --reps 100 $SWEEP_ARGS >> gpurun_out/sweep.txt 2>&1
  if [ -n "$SWEEP_SIZES" ]; then
    SVDLUT_LIB=$f timeout 120 python tools/kbench.py --variant 0 --reps 50 --only smooth --h 1080 --w 1920 >> gpurun_out/sweep.txt 2>&1
    SVDLUT_LIB=$f timeout 120 python tools/kbench.py --variant 0 --reps 20 --only smooth --h 4320 --w 7680 >> gpurun_out/sweep.txt 2>&1
  fi
done
