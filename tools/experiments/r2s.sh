set -u
OUT=gpurun_out/r2s
mkdir -p $OUT
export FFTPIM_K4_RUNS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "run_encoded" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
export FFTPIM_K4_OVERLAP=0
timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/c4_w24s2.jsonl 2> $OUT/c4_w24s2.err; echo "c4 w24s2 rc=$?"
for v in w16s3 w12s4 w20s2; do
  FFTPIM_LIB=$PWD/paper_2312_02376_b200/lib/variants/libfftpim_$v.so timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/c4_$v.jsonl 2> $OUT/c4_$v.err; echo "c4 $v rc=$?"
done
export FFTPIM_K4_OVERLAP=1
timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/c4_w24s2_ovl.jsonl 2> $OUT/c4_w24s2_ovl.err; echo "c4 w24s2 ovl rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
export FFTPIM_NO_GRAPHS=1
export FFTPIM_K4_OVERLAP=0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_corr_runs" -s 2 -c 1 -o $OUT/k4runs $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
