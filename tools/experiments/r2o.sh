set -u
OUT=gpurun_out/r2o
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests.log
timeout 900 python bench.py > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err; echo "bench c4 rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
export FFTPIM_NO_GRAPHS=1
if timeout 600 $CMD > $OUT/plain.log 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
fi
