mkdir -p gpurun_out/s7
L=paper_2312_02376_b200/lib
for c in 2 4 3; do
 for v in base pf3 default; do
  if [ $v = default ]; then lib=$L/libfftpim.so; else lib=$L/variants/libfftpim_$v.so; fi
  FFTPIM_LIB=$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s7/c${c}_$v.jsonl 2> gpurun_out/s7/c${c}_$v.err
  echo "c$c $v rc=$?"
 done
done
