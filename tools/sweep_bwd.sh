python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/sweep_bwd.txt
for f in paper_2508_16121_b200/_lib/variants/lib*.so; do
  echo "== $f" >> gpurun_out/sweep_bwd.txt
  SVDLUT_LIB=$f timeout 200 python tools/bwdbench.py >> gpurun_out/sweep_bwd.txt 2>&1
done
