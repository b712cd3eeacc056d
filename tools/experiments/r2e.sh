set -u
OUT=gpurun_out/r2e
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "point_paths" > $OUT/test_parity.log 2>&1; echo "parity rc=$?"; tail -2 $OUT/test_parity.log
FFTPIM_K1=lines_smem timeout 600 python bench.py --no-cpu-baseline --steps 5 > $OUT/bench_c4_smem.jsonl 2> $OUT/bench_c4_smem.err; echo "bench c4 smem rc=$?"
FFTPIM_K1=lines_smem FFTPIM_NO_GRAPHS=1 timeout 600 ncu --set full --clock-control none -k regex:"k_k1_lines" -s 1 -c 1 -o $OUT/c4_smem python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_smem.log 2>&1; echo "ncu smem rc=$?"
