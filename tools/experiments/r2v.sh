set -u
OUT=gpurun_out/r2v
mkdir -p $OUT
FFTPIM_K4_C16=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -q -x -k "c16 or offsets16 or small_case_parity_single or source_ordered" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
FFTPIM_K4_C16=1 timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/c4_o16.jsonl 2> $OUT/c4_o16.err; echo "c4 o16 rc=$?"
timeout 900 python bench.py --no-cpu-baseline --steps 5 > $OUT/c4_base.jsonl 2> $OUT/c4_base.err; echo "c4 base rc=$?"
FFTPIM_K4_C16=1 timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 > $OUT/c3_o16.jsonl 2> $OUT/c3_o16.err; echo "c3 o16 rc=$?"
timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 > $OUT/c3_base.jsonl 2> $OUT/c3_base.err; echo "c3 base rc=$?"
