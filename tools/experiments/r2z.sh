set -u
OUT=gpurun_out/r2z
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_paths.py -q -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_pf.jsonl 2> $OUT/c4_pf.err; echo "c4 pf rc=$?"
FFTPIM_LIB=$PWD/paper_2312_02376_b200/lib/variants/libfftpim_nopf.so timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_nopf.jsonl 2> $OUT/c4_nopf.err; echo "c4 nopf rc=$?"
timeout 900 python bench.py --config 5 --per-excitation --no-cpu-baseline --steps 10 > $OUT/c5pe_pf.jsonl 2> $OUT/c5pe_pf.err; echo "c5pe pf rc=$?"
FFTPIM_LIB=$PWD/paper_2312_02376_b200/lib/variants/libfftpim_nopf.so timeout 900 python bench.py --config 5 --per-excitation --no-cpu-baseline --steps 10 > $OUT/c5pe_nopf.jsonl 2> $OUT/c5pe_nopf.err; echo "c5pe nopf rc=$?"
