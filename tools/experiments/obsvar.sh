mkdir -p gpurun_out/s29
L=paper_2312_02376_b200/lib
for v in lpo1 lpo2 lpo2m6; do
  if [ $v = default ]; then lib=$L/libfftpim.so; else lib=$L/variants/libfftpim_$v.so; fi
  for c in 2 4; do
    FFTPIM_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s29/c${c}_$v.jsonl 2>&1
  done
  FFTPIM_LIB=$lib timeout 600 python bench.py --config 5 --per-excitation --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s29/c5pe_$v.jsonl 2>&1
  echo "$v done"
done
