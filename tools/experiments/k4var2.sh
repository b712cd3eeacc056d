mkdir -p gpurun_out/s36
L=paper_2312_02376_b200/lib
for v in default r1 c2; do
  if [ $v = default ]; then lib=$L/libfftpim.so; else lib=$L/variants/libfftpim_$v.so; fi
  for c in 3 1; do FFTPIM_LIB=$lib timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s36/c${c}_$v.jsonl 2>&1; done
  if [ $v != r1 ]; then
    FFTPIM_LIB=$lib timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s36/c4_$v.jsonl 2>&1
    FFTPIM_LIB=$lib timeout 900 python bench.py --config 5 --per-excitation --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s36/c5pe_$v.jsonl 2>&1
    FFTPIM_LIB=$lib timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/s36/c2_$v.jsonl 2>&1
  fi
  echo $v done
done
