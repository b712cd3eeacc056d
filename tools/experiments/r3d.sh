# Round 2 (session 4): K1 line sweep with R = 2 z lines per thread (more resident warps) against the default R = 4.
set -u
OUT=gpurun_out/r3d
mkdir -p $OUT
V=$PWD/paper_2312_02376_b200/lib/variants
for v in k1r2a k1r2b k1r2c; do
  FFTPIM_LIB=$V/libfftpim_$v.so timeout 600 python -m pytest tests/test_gpu_paths.py -q -x -k "k1_ell" > $OUT/tests_$v.log 2>&1; echo "tests $v rc=$?"; tail -2 $OUT/tests_$v.log
  FFTPIM_LIB=$V/libfftpim_$v.so timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_$v.jsonl 2> $OUT/c4_$v.err; echo "c4 $v rc=$?"
done
timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_default.jsonl 2> $OUT/c4_default.err; echo "c4 default rc=$?"
python tools/showbench.py $OUT/c4_*.jsonl
