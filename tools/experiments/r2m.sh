set -u
OUT=gpurun_out/r2m
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "source_ordered or subset" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
for v in "FFTPIM_K4_SORT=1" "FFTPIM_K4_SORT=0"; do
  tag=$(echo "$v" | tr ' =/' '___')
  env $v timeout 600 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_$tag.jsonl 2> $OUT/c4_$tag.err; echo "c4 $v rc=$?"
  env $v timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 > $OUT/c3_$tag.jsonl 2> $OUT/c3_$tag.err; echo "c3 $v rc=$?"
done
timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 5 --per-excitation > $OUT/c5pe.jsonl 2> $OUT/c5pe.err; echo "c5pe rc=$?"
