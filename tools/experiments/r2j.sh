set -u
OUT=gpurun_out/r2j
mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err; echo "bench c4 rc=$?"
timeout 300 python bench.py --config 2 --no-cpu-baseline > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err; echo "bench c2 rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
