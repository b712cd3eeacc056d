#!/usr/bin/env bash
# Final round-2 evidence on one B200 (gpurun, repo root): the whole GPU test suite, smoke(), the default bench line and the
# reference arm with the driver's flags, the ncu launch list of the default bench command and a --set full capture of one
# evaluation's kernels.  Each ncu pass runs after the same command exited 0 without ncu.  Outputs: gpurun_out/final/.
set -u
OUT=${OUT:-gpurun_out/final}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit --format=csv > $OUT/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
( time timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err ) 2> $OUT/bench_c4.time; echo "bench c4 rc=$?"
( time timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref_c4.jsonl 2> $OUT/ref_c4.err ) 2> $OUT/ref_c4.time; echo "ref c4 rc=$?"
timeout 900 python bench.py --config 2 > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err; echo "bench c2 rc=$?"
export FFTPIM_NO_GRAPHS=1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
if timeout 600 $CMD > $OUT/plain.log 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file $OUT/c4_launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"k_corr_tiles|k_k1_lines|k_observers|k_fft_reg|k_far_project|k_permute_q" -s 9 -c 10 \
    -f -o /tmp/c4_full $CMD > $OUT/ncu_c4_full.log 2>&1; echo "ncu c4 full rc=$?"
  ncu -i /tmp/c4_full.ncu-rep --page raw --csv > $OUT/c4_full_raw.csv 2>/dev/null
fi
cat $OUT/bench_c4.time $OUT/ref_c4.time
