# Round 2 (session 4): FP64 pipe probe; edge-case tests; far projection at 3 blocks per SM / one-wave chunks A/B.
set -u
OUT=gpurun_out/r3c
mkdir -p $OUT
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_probe.cu -o /tmp/fp64_probe && timeout 120 /tmp/fp64_probe > $OUT/fp64_probe.txt 2>&1; cat $OUT/fp64_probe.txt
timeout 1500 python -m pytest tests/test_gpu_edge_cases.py tests/test_gpu_paths.py tests/test_gpu_sharding.py tests/test_gpu_parity.py -q -x -k "edge or far_windows or point_paths or slab_group_emulated or slab_group_dynamic or w8" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/tests.log
for c in 4 3 5; do
  X=""; [ $c = 5 ] && X="--per-excitation"
  timeout 900 python bench.py --config $c $X --no-cpu-baseline --steps 10 > $OUT/c${c}_cap256.jsonl 2> $OUT/c${c}_cap256.err; echo "c$c cap256 rc=$?"
  FFTPIM_FAR_CAP=400 timeout 900 python bench.py --config $c $X --no-cpu-baseline --steps 10 > $OUT/c${c}_cap400.jsonl 2> $OUT/c${c}_cap400.err; echo "c$c cap400 rc=$?"
done
python tools/showbench.py $OUT/c*_cap*.jsonl
