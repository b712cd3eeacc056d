mkdir -p gpurun_out/s10
L=paper_2312_02376_b200/lib
for c in 2 4; do
 for v in k1old default; do
  if [ $v = default ]; then lib=$L/libfftpim.so; else lib=$L/variants/libfftpim_$v.so; fi
  FFTPIM_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s10/c${c}_$v.jsonl 2> gpurun_out/s10/c${c}_$v.err
  echo "c$c $v rc=$?"
 done
done
FFTPIM_LIB=$L/libfftpim.so timeout 600 python bench.py --config 5 --per-excitation --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s10/c5pe.jsonl 2>&1; echo c5pe rc=$?
