set -u
OUT=gpurun_out/r2h
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "register_fft" > $OUT/test_fft.log 2>&1; echo "fft tests rc=$?"; tail -2 $OUT/test_fft.log
export FFTPIM_K1=lines_smem FFTPIM_OBS=tile FFTPIM_FAR=win
timeout 600 python bench.py --no-cpu-baseline --steps 10 > $OUT/bench_c4_r8.jsonl 2> $OUT/bench_c4_r8.err; echo "bench c4 r8 rc=$?"
FFTPIM_FFT_R8=0 timeout 600 python bench.py --no-cpu-baseline --steps 10 > $OUT/bench_c4_e32.jsonl 2> $OUT/bench_c4_e32.err; echo "bench c4 e32 rc=$?"
FFTPIM_NO_GRAPHS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fft_r8x3" -s 3 -c 3 -o $OUT/c4_r8 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_r8.log 2>&1; echo "ncu rc=$?"
