mkdir -p gpurun_out/s30
for cfg in "8 1" "4 2" "4 3" "2 4" "6 2"; do
  set -- $cfg
  for c in 2 4; do
    FFTPIM_FAR_WARPS=$1 FFTPIM_FAR_BPS=$2 timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s30/c${c}_w$1_b$2.jsonl 2>&1
  done
  FFTPIM_FAR_WARPS=$1 FFTPIM_FAR_BPS=$2 timeout 600 python bench.py --config 5 --per-excitation --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s30/c5pe_w$1_b$2.jsonl 2>&1
done
echo done
