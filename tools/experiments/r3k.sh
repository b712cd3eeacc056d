# Fused x stage with the spectrum loads issued right after the exchange barrier (FFT_SPEC_EARLY=1) against the previous order.
set -u
OUT=gpurun_out/r3k
mkdir -p $OUT
V=$PWD/paper_2312_02376_b200/lib/variants
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x -k "register_fft or baseline_config_parity or small_case_parity" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
for rep in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_early_$rep.jsonl 2> $OUT/c4_early_$rep.err; echo "early rc=$?"
  FFTPIM_LIB=$V/libfftpim_specoff.so timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_late_$rep.jsonl 2> $OUT/c4_late_$rep.err; echo "late rc=$?"
done
for rep in 1 2; do
  timeout 900 python bench.py --config 2 --no-cpu-baseline > $OUT/c2_early_$rep.jsonl 2> $OUT/c2_early_$rep.err
  FFTPIM_LIB=$V/libfftpim_specoff.so timeout 900 python bench.py --config 2 --no-cpu-baseline > $OUT/c2_late_$rep.jsonl 2> $OUT/c2_late_$rep.err
done
timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 10 > $OUT/c3_early.jsonl 2> $OUT/c3_early.err
FFTPIM_LIB=$V/libfftpim_specoff.so timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 10 > $OUT/c3_late.jsonl 2> $OUT/c3_late.err
python tools/showbench.py $OUT/c*.jsonl | grep -v fp64
