set -u
OUT=gpurun_out/r2k
mkdir -p $OUT
export FFTPIM_NO_GRAPHS=1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/c4_launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_corr_tiles|k_k1_lines|k_observers_tile|k_far_project_win|k_fft_reg|k_permute" -s 12 -c 8 -o $OUT/c4_full $CMD > $OUT/ncu_full.log 2>&1; echo "full rc=$?"
