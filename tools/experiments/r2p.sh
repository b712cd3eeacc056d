set -u
OUT=gpurun_out/r2p
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "run_encoded or source_ordered or subset" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_runs.jsonl 2> $OUT/c4_runs.err; echo "c4 runs rc=$?"
FFTPIM_K4_RUNS=0 timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_noruns.jsonl 2> $OUT/c4_noruns.err; echo "c4 noruns rc=$?"
timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 > $OUT/c3_runs.jsonl 2> $OUT/c3_runs.err; echo "c3 runs rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
export FFTPIM_NO_GRAPHS=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_corr_runs" -s 2 -c 1 -o $OUT/k4runs $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
