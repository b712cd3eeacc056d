cd $GRAFT_REPO_ROOT
for env in "" "FFTPIM_CORR_BLOCKS=148" "FFTPIM_CORR_BLOCKS=296" "FFTPIM_CORR_BLOCKS=185" "FFTPIM_CORR_BLOCKS=259" "FFTPIM_K4_GATE=1" "FFTPIM_FAR_WARPS=4" "FFTPIM_FAR_WARPS=16" "FFTPIM_OBS_FUSED=1" "FFTPIM_K1_ORIG=0"; do
  for rep in 1 2; do
    v=$(env $env python bench.py --no-cpu-baseline --steps 200 --warmup 20 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), d['roofline']['kernel_ms']*1000)")
    echo "[$env] $v"
  done
done
