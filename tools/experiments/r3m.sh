# Observer tile pass: far-grid copy with four loads in flight per thread, against the previous library.
set -u
OUT=gpurun_out/r3m
mkdir -p $OUT
V=$PWD/paper_2312_02376_b200/lib/variants
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -q -x -k "point_paths or edge or baseline_config_subset" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
for rep in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_new_$rep.jsonl 2> $OUT/c4_new_$rep.err
  FFTPIM_LIB=$V/libfftpim_prev.so timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_old_$rep.jsonl 2> $OUT/c4_old_$rep.err
done
python tools/showbench.py $OUT/c*.jsonl | grep stages | sed 's/.*observers/observers/'
