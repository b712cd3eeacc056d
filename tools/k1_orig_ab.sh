# A/B of the K1 charge-order switch (FFTPIM_K1_ORIG) on C1 and C2, alternating runs
cd $GRAFT_REPO_ROOT
for cfg in 2 1; do
  for rep in 1 2 3; do
    for v in 1 0; do
      r=$(FFTPIM_K1_ORIG=$v python bench.py --config $cfg --no-cpu-baseline --steps 300 --warmup 20 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us  e2e', '%.3g' % d['e2e']['value'])")
      echo "C$cfg K1_ORIG=$v $r"
    done
  done
done
