# Source-level ncu pages (SASS with stall samples) of the C4 x-stage FFT, the K1 line sweep and the observer tile pass.
set -u
OUT=gpurun_out/r3i
mkdir -p $OUT
export FFTPIM_NO_GRAPHS=1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
for spec in "k_fft_reg:2:fftx" "k_k1_lines:0:k1" "k_observers_tile:0:obs"; do
  K=${spec%%:*}; rest=${spec#*:}; S=${rest%%:*}; N=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -f -o /tmp/$N $CMD > $OUT/ncu_$N.log 2>&1; echo "ncu $N rc=$?"
  ncu -i /tmp/$N.ncu-rep --page source --csv > $OUT/${N}_source.csv 2>/dev/null
  ncu -i /tmp/$N.ncu-rep --page raw --csv > $OUT/${N}_raw.csv 2>/dev/null
done
ls -la $OUT
