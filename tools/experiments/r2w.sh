set -u
OUT=gpurun_out/r2w
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_sweep.py -q -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 5 > $OUT/c5_rows2.jsonl 2> $OUT/c5_rows2.err; echo "c5 rows2 rc=$?"
FFTPIM_SWEEP_ROWS2=0 timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 5 > $OUT/c5_rows1.jsonl 2> $OUT/c5_rows1.err; echo "c5 rows1 rc=$?"
timeout 900 python bench.py --config 4 --batch 64 --no-cpu-baseline --steps 3 > $OUT/c4_b64_rows2.jsonl 2> $OUT/c4_b64_rows2.err; echo "c4 b64 rows2 rc=$?"
FFTPIM_SWEEP_ROWS2=0 timeout 900 python bench.py --config 4 --batch 64 --no-cpu-baseline --steps 3 > $OUT/c4_b64_rows1.jsonl 2> $OUT/c4_b64_rows1.err; echo "c4 b64 rows1 rc=$?"
