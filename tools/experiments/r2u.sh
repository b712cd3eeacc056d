set -u
OUT=gpurun_out/r2u
mkdir -p $OUT
export FFTPIM_K4_RUNS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "run_encoded" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
FFTPIM_K4_OVERLAP=0 timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/c4_rl_seq.jsonl 2> $OUT/c4_rl_seq.err; echo "c4 rl seq rc=$?"
FFTPIM_K4_OVERLAP=1 timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/c4_rl_ovl.jsonl 2> $OUT/c4_rl_ovl.err; echo "c4 rl ovl rc=$?"
FFTPIM_K4_OVERLAP=1 FFTPIM_K4A_BLOCKS=296 FFTPIM_K4B_BLOCKS=0 timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/c4_rl_ovl296.jsonl 2> $OUT/c4_rl_ovl296.err; echo "c4 rl ovl296 rc=$?"
FFTPIM_K4_OVERLAP=1 FFTPIM_K4_RUNS_KERNEL=bulk FFTPIM_LIB=$PWD/paper_2312_02376_b200/lib/variants/libfftpim_w16s2.so timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/c4_bulk_ovl.jsonl 2> $OUT/c4_bulk_ovl.err; echo "c4 bulk ovl rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
export FFTPIM_NO_GRAPHS=1
export FFTPIM_K4_OVERLAP=0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_corr_rl" -s 2 -c 1 -o $OUT/k4rl $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
