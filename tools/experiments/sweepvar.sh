mkdir -p gpurun_out/s39
L=paper_2312_02376_b200/lib
timeout 600 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/s39/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s39/pytest.log
for v in default pf_m2 nopf; do
  if [ $v = default ]; then lib=$L/libfftpim.so; else lib=$L/variants/libfftpim_$v.so; fi
  FFTPIM_LIB=$lib timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s39/c5_$v.jsonl 2> gpurun_out/s39/c5_$v.err
  FFTPIM_LIB=$lib timeout 600 python tools/batch_bench.py --config 5 --batch 64 --reps 2 > gpurun_out/s39/b5_$v.json 2>&1; echo "$v $(tail -1 gpurun_out/s39/b5_$v.json | cut -c60-140)"
done
