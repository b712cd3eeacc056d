set -u
OUT=gpurun_out/r2n
mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests.log
timeout 900 python bench.py > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err; echo "bench c4 rc=$?"
timeout 900 python bench.py --impl reference > $OUT/ref_c4.jsonl 2> $OUT/ref_c4.err; echo "ref c4 rc=$?"
