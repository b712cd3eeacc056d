#!/usr/bin/env bash
# Round-2 evidence on one B200 (run through gpurun from the repo root): the GPU
# test suite, smoke(), the default (C4) bench line with its composed CPU baseline,
# the reference arm, bench lines for the other configs, the ncu launch list of the
# default bench command, `--set full` captures of the evaluation kernels (C4),
# the C3 K4 and the C5 sweep K4 (the .ncu-rep files stay in /tmp on the box; their raw
# pages come back as CSV).  Each ncu pass runs only after the same command exited 0 without ncu.
# Outputs land in gpurun_out/round2/.
set -u
OUT=gpurun_out/round2
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit --format=csv > $OUT/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err; echo "bench c4 rc=$?"
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref_c4.jsonl 2> $OUT/ref_c4.err; echo "ref c4 rc=$?"
for c in 1 2 3 5; do
  timeout 1200 python bench.py --config $c > $OUT/bench_c$c.jsonl 2> $OUT/bench_c$c.err; echo "bench c$c rc=$?"
done
timeout 900 python bench.py --config 5 --per-excitation --no-cpu-baseline > $OUT/bench_c5pe.jsonl 2> $OUT/bench_c5pe.err; echo "bench c5pe rc=$?"
timeout 900 python bench.py --config 4 --batch 64 --no-cpu-baseline --steps 3 > $OUT/bench_c4_b64.jsonl 2> $OUT/bench_c4_b64.err; echo "bench c4 b64 rc=$?"
timeout 900 python bench.py --config 2 --impl reference --steps 3 --warmup 1 > $OUT/ref_c2.jsonl 2> $OUT/ref_c2.err; echo "ref c2 rc=$?"
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
CMD3="python bench.py --config 3 --steps 1 --warmup 2 --no-cpu-baseline"
# C3 holds 172 GB: a multi-pass --set full capture cannot save/restore device memory, so
# the single-pass launch list (time + DRAM bytes per launch) stands in for it
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 300 --csv --log-file $OUT/c3_launches.csv $CMD3 > $OUT/ncu_c3_launches.log 2>&1; echo "ncu c3 launches rc=$?"
CMD5="python bench.py --config 5 --steps 1 --warmup 2 --no-cpu-baseline"
unset FFTPIM_NO_GRAPHS
timeout 1200 ncu --set full --clock-control none -k regex:"k_corr_sweep" -s 1 -c 1 \
    -f -o /tmp/c5_sweep $CMD5 > $OUT/ncu_c5_sweep.log 2>&1; echo "ncu c5 sweep rc=$?"
ncu -i /tmp/c5_sweep.ncu-rep --page raw --csv > $OUT/c5_sweep_raw.csv 2>/dev/null
# compute-sanitizer is closed on this pool (gpurun refuses it): not run.
