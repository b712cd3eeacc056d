set -u
OUT=gpurun_out/r2y
mkdir -p $OUT
export FFTPIM_SWEEP_ASYNC=0
FFTPIM_SWEEP_ROWS2=1 timeout 1500 python -m pytest tests/test_gpu_sweep.py -q -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
FFTPIM_SWEEP_ROWS2=1 timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 5 > $OUT/c5_rows2.jsonl 2> $OUT/c5_rows2.err; echo "c5 rows2 rc=$?"
FFTPIM_SWEEP_ROWS2=1 FFTPIM_LIB=$PWD/paper_2312_02376_b200/lib/variants/libfftpim_r2m3.so timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 5 > $OUT/c5_rows2_m3.jsonl 2> $OUT/c5_rows2_m3.err; echo "c5 rows2 m3 rc=$?"
timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 5 > $OUT/c5_base.jsonl 2> $OUT/c5_base.err; echo "c5 base rc=$?"
FFTPIM_SWEEP_ROWS2=1 timeout 900 python bench.py --config 4 --batch 64 --no-cpu-baseline --steps 3 > $OUT/c4_b64_rows2.jsonl 2> $OUT/c4_b64_rows2.err; echo "c4 b64 rows2 rc=$?"
