# Far projection with the next batch's loads in flight and the observer tile pass with the first observer's position
# loaded before the tile loads, against the previous library.
set -u
OUT=gpurun_out/r3l
mkdir -p $OUT
V=$PWD/paper_2312_02376_b200/lib/variants
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_sharding.py tests/test_gpu_edge_cases.py tests/test_gpu_random.py -q -x -k "point_paths or far_windows or slab_group or edge or baseline_config_subset or random" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
for rep in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_new_$rep.jsonl 2> $OUT/c4_new_$rep.err; echo "new rc=$?"
  FFTPIM_LIB=$V/libfftpim_prev.so timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_old_$rep.jsonl 2> $OUT/c4_old_$rep.err; echo "old rc=$?"
done
timeout 900 python bench.py --config 5 --per-excitation --no-cpu-baseline --steps 10 > $OUT/c5_new.jsonl 2> $OUT/c5_new.err
FFTPIM_LIB=$V/libfftpim_prev.so timeout 900 python bench.py --config 5 --per-excitation --no-cpu-baseline --steps 10 > $OUT/c5_old.jsonl 2> $OUT/c5_old.err
timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 10 > $OUT/c3_new.jsonl 2> $OUT/c3_new.err
FFTPIM_LIB=$V/libfftpim_prev.so timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 10 > $OUT/c3_old.jsonl 2> $OUT/c3_old.err
python tools/showbench.py $OUT/c*.jsonl | grep -v fp64
