set -u
OUT=gpurun_out/r2c
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "k1" > $OUT/test_k1.log 2>&1; echo "k1 tests rc=$?"; tail -2 $OUT/test_k1.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "point_paths or subset" > $OUT/test_parity.log 2>&1; echo "parity rc=$?"; tail -2 $OUT/test_parity.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err; echo "bench c4 rc=$?"
FFTPIM_K1=lines_smem timeout 600 python bench.py --no-cpu-baseline --steps 5 > $OUT/bench_c4_smem.jsonl 2> $OUT/bench_c4_smem.err; echo "bench c4 smem rc=$?"
FFTPIM_K1=lines FFTPIM_OBS=pos timeout 300 python bench.py --config 2 --no-cpu-baseline > $OUT/bench_c2_lines.jsonl 2> $OUT/bench_c2_lines.err; echo "bench c2 lines rc=$?"
for c in 3 5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > $OUT/bench_c$c.jsonl 2> $OUT/bench_c$c.err; echo "bench c$c rc=$?"; done
