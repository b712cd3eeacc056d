set -u
OUT=gpurun_out/r2g
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "point_paths" > $OUT/test_parity.log 2>&1; echo "parity rc=$?"; tail -2 $OUT/test_parity.log
export FFTPIM_K1=lines_smem FFTPIM_OBS=tile FFTPIM_FAR=win
timeout 600 python bench.py --no-cpu-baseline --steps 5 > $OUT/bench_c4_new.jsonl 2> $OUT/bench_c4_new.err; echo "bench c4 new rc=$?"
timeout 300 python bench.py --config 2 --no-cpu-baseline > $OUT/bench_c2_new.jsonl 2> $OUT/bench_c2_new.err; echo "bench c2 new rc=$?"
FFTPIM_NO_GRAPHS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_k1_lines|k_observers_tile|k_far_project_win|k_far_windows" -s 4 -c 4 -o $OUT/c4_new python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_new.log 2>&1; echo "ncu rc=$?"
