set -u
OUT=gpurun_out/r2x
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_sweep.py -q -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 5 > $OUT/c5_async.jsonl 2> $OUT/c5_async.err; echo "c5 async rc=$?"
for v in d4m3 d12m1; do
FFTPIM_LIB=$PWD/paper_2312_02376_b200/lib/variants/libfftpim_$v.so timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 5 > $OUT/c5_$v.jsonl 2> $OUT/c5_$v.err; echo "c5 $v rc=$?"
done
timeout 900 python bench.py --config 4 --batch 64 --no-cpu-baseline --steps 3 > $OUT/c4_b64_async.jsonl 2> $OUT/c4_b64_async.err; echo "c4 b64 async rc=$?"
timeout 900 python bench.py --batch 64 --config 2 --no-cpu-baseline --steps 10 --warmup 3 > $OUT/c2_b64_async.jsonl 2> $OUT/c2_b64_async.err; echo "c2 b64 async rc=$?"
