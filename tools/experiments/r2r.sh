set -u
OUT=gpurun_out/r2r
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "run_encoded or subset" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
FFTPIM_K4_OVERLAP=0 timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_runs_seq.jsonl 2> $OUT/c4_runs_seq.err; echo "c4 runs seq rc=$?"
timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_runs_ovl.jsonl 2> $OUT/c4_runs_ovl.err; echo "c4 runs ovl rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
export FFTPIM_NO_GRAPHS=1
export FFTPIM_K4_OVERLAP=0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_corr_runs" -s 2 -c 1 -o $OUT/k4runs $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
