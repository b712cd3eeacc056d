#!/usr/bin/env bash
# Short evidence refresh (C2 bench + reference arm, C1/C4 lines, C2 ncu launch list + full capture)
set -u
OUT=gpurun_out/round
mkdir -p $OUT
python bench.py > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err; echo "bench c2 rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.jsonl 2> $OUT/bench_ref.err; echo "ref rc=$?"
for c in 1 4; do
  python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_c$c.jsonl 2> $OUT/bench_c$c.err; echo "bench c$c rc=$?"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
export FFTPIM_NO_GRAPHS=1
if timeout 300 $CMD > $OUT/plain.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_corr_tiles|k_k1_spmv|k_observers|k_fft_reg|k_far_project" -s 12 -c 12 \
    -o $OUT/full $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
