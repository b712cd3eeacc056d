# Round 2 (session 4): edge-case parity tests, far projection v2 (plan-time windows, ballot runs) A/B at C4/C3/C5,
# ncu --set full of the far projection kernels with the source page.
set -u
OUT=gpurun_out/r3a
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_edge_cases.py tests/test_gpu_paths.py -q -x -k "edge or far_windows or domain or two_points or single or one_source or nodes or stencils or boundary or face or one_cell or reciprocity" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/tests.log
for c in 4 3 5; do
  X=""; [ $c = 5 ] && X="--per-excitation"
  timeout 900 python bench.py --config $c $X --no-cpu-baseline --steps 10 > $OUT/c${c}_win2.jsonl 2> $OUT/c${c}_win2.err; echo "c$c win2 rc=$?"
  FFTPIM_FAR_WIN2=0 timeout 900 python bench.py --config $c $X --no-cpu-baseline --steps 10 > $OUT/c${c}_win1.jsonl 2> $OUT/c${c}_win1.err; echo "c$c win1 rc=$?"
done
python tools/showbench.py $OUT/c*_win*.jsonl
export FFTPIM_NO_GRAPHS=1
CMD="python bench.py --steps 1 --warmup 2 --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_far_project_win" -s 1 -c 1 \
    -f -o /tmp/far2 $CMD > $OUT/ncu_far2.log 2>&1; echo "ncu far2 rc=$?"
ncu -i /tmp/far2.ncu-rep --page raw --csv > $OUT/far2_raw.csv 2>/dev/null
ncu -i /tmp/far2.ncu-rep --page source --csv > $OUT/far2_source.csv 2>/dev/null
FFTPIM_FAR_WIN2=0 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_far_project_win" -s 1 -c 1 \
    -f -o /tmp/far1 $CMD > $OUT/ncu_far1.log 2>&1; echo "ncu far1 rc=$?"
ncu -i /tmp/far1.ncu-rep --page raw --csv > $OUT/far1_raw.csv 2>/dev/null
ncu -i /tmp/far1.ncu-rep --page source --csv > $OUT/far1_source.csv 2>/dev/null
ls -la $OUT
