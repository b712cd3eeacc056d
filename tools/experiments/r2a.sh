set -u
OUT=gpurun_out/r2a
mkdir -p $OUT
nproc > $OUT/nproc.txt
python bench.py > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err; echo "bench c4 rc=$?"
python bench.py --impl reference > $OUT/ref_c4.jsonl 2> $OUT/ref_c4.err; echo "ref c4 rc=$?"
python bench.py --config 2 > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err; echo "bench c2 rc=$?"
