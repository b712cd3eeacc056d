set -u
OUT=gpurun_out/r2i
mkdir -p $OUT
python tools/bw_probe.py > $OUT/bw.txt 2>&1; cat $OUT/bw.txt
for c in 3 5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --per-excitation > $OUT/bench_c${c}_old.jsonl 2> $OUT/bench_c${c}_old.err; echo "c$c old rc=$?"
  FFTPIM_K1=lines_smem FFTPIM_OBS=tile FFTPIM_FAR=win timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --per-excitation > $OUT/bench_c${c}_new.jsonl 2> $OUT/bench_c${c}_new.err; echo "c$c new rc=$?"
done
FFTPIM_OBS=tile FFTPIM_FAR=win timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 > $OUT/bench_c3_ellk1.jsonl 2> $OUT/bench_c3_ellk1.err; echo "c3 ell-k1 rc=$?"
