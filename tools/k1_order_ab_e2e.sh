# A/B: two K1 index orders (default) vs one caller-order operator (FFTPIM_K1_ONE_ORDER=1), C2 and C1
cd $GRAFT_REPO_ROOT
for cfg in 2; do
  for rep in 1 2 3 4 5; do
    for v in "" "FFTPIM_K1_ONE_ORDER=1"; do
      r=$(env $v python bench.py --config $cfg --no-cpu-baseline --steps 2000 --warmup 20 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us  e2e', '%.3g' % d['e2e']['value'], 'rel', d.get('rel_l2_vs_reference'))")
      echo "C$cfg [$v] $r"
    done
  done
done
