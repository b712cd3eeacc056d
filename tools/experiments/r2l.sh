set -u
OUT=gpurun_out/r2l
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_boundary.py -x -q -k "k4_16bit or boundary or retained or zone or cache or provider" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
for v in "FFTPIM_K4_C16=0" "FFTPIM_K4_C16=1" "FFTPIM_K4_C16=0 FFTPIM_CONCURRENT_MAX=1000000000000" "FFTPIM_K4_C16=0 FFTPIM_LIB=paper_2312_02376_b200/lib/variants/libfftpim_nogather.so"; do
  tag=$(echo "$v" | tr ' =/' '___' | cut -c1-60)
  env $v timeout 600 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_$tag.jsonl 2> $OUT/c4_$tag.err; echo "c4 $v rc=$?"
done
FFTPIM_K4_C16=1 timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 > $OUT/c3_c16.jsonl 2> $OUT/c3_c16.err; echo "c3 c16 rc=$?"
FFTPIM_K4_C16=0 timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 > $OUT/c3_c32.jsonl 2> $OUT/c3_c32.err; echo "c3 c32 rc=$?"
