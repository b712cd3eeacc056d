# Round 2 (session 4): far projection with four points per warp step (k_far_project_win4) against the general kernel.
set -u
OUT=gpurun_out/r3e
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_sharding.py tests/test_gpu_edge_cases.py -q -x -k "far_windows or point_paths or slab_group_emulated or slab_group_dynamic or w8 or edge" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/tests.log
for rep in 1 2; do
for c in 4 5 3; do
  X=""; [ $c = 5 ] && X="--per-excitation"
  timeout 900 python bench.py --config $c $X --no-cpu-baseline --steps 10 > $OUT/c${c}_win4_$rep.jsonl 2> $OUT/c${c}_win4_$rep.err; echo "c$c win4 rc=$?"
  FFTPIM_FAR_WIN4=0 timeout 900 python bench.py --config $c $X --no-cpu-baseline --steps 10 > $OUT/c${c}_win1_$rep.jsonl 2> $OUT/c${c}_win1_$rep.err; echo "c$c win1 rc=$?"
done
done
python tools/showbench.py $OUT/c*_win*.jsonl | grep -v fp64
