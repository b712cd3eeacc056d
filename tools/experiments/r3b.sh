# Round 2 (session 4): edge-case parity tests, persistent copy pool A/B on the pageable host entry (C4),
# filtered ncu launch lists of the C3 and C5 evaluation kernels, compute-sanitizer probe.
set -u
OUT=gpurun_out/r3b
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_edge_cases.py tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x -k "edge or far_windows or pageable or host_entries or concurrent" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/tests.log
timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_pool.jsonl 2> $OUT/c4_pool.err; echo "c4 pool rc=$?"
FFTPIM_LIB=$PWD/paper_2312_02376_b200/lib/variants/libfftpim_prepool.so timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_prepool.jsonl 2> $OUT/c4_prepool.err; echo "c4 prepool rc=$?"
FFTPIM_HOST_COPY_THREADS=16 timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_pool16.jsonl 2> $OUT/c4_pool16.err; echo "c4 pool16 rc=$?"
FFTPIM_HOST_COPY_THREADS=4 timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_pool4.jsonl 2> $OUT/c4_pool4.err; echo "c4 pool4 rc=$?"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r3b/c4_*.jsonl')):
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l); print(f, 'ms=%.3f'%d['ms_per_step'], 'e2e=%.4g'%d['e2e']['value'], 'pageable=%.4g'%d['e2e_pageable']['value'])
PY
nproc
export FFTPIM_NO_GRAPHS=1
K='regex:k_corr_tiles|k_k1_|k_observers|k_fft_|k_far_|k_permute_q|k_corr_sweep'
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "$K" -c 60 --csv --log-file $OUT/c3_eval_launches.csv python bench.py --config 3 --steps 1 --warmup 2 --no-cpu-baseline > $OUT/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "$K" -c 60 --csv --log-file $OUT/c5pe_eval_launches.csv python bench.py --config 5 --per-excitation --steps 1 --warmup 2 --no-cpu-baseline > $OUT/ncu_c5pe.log 2>&1; echo "ncu c5pe rc=$?"
unset FFTPIM_NO_GRAPHS
timeout 600 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitizer.log 2>&1; echo "sanitizer rc=$?"; tail -5 $OUT/sanitizer.log
