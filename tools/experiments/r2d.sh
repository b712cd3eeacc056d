set -u
OUT=gpurun_out/r2d
mkdir -p $OUT
export FFTPIM_NO_GRAPHS=1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_k1_lines_g|k_observers_pos|k_far_project|k_fft_reg" -s 4 -c 6 -o $OUT/c4_g $CMD > $OUT/ncu_g.log 2>&1; echo "ncu g rc=$?"
FFTPIM_K1=lines_smem timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_k1_lines" -s 1 -c 1 -o $OUT/c4_smem $CMD > $OUT/ncu_smem.log 2>&1; echo "ncu smem rc=$?"
