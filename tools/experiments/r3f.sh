# Round 2 (session 4): observer tile pass at 3 / 5 blocks per SM (register budget 80 / 48), L = 512 register FFT with in-place
# 32-point DFTs at 3 blocks per SM (FFTPIM_FFT_IP=1), against the defaults; C4, 10 steps each, twice.
set -u
OUT=gpurun_out/r3f
mkdir -p $OUT
V=$PWD/paper_2312_02376_b200/lib/variants
for rep in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_default_$rep.jsonl 2> $OUT/c4_default_$rep.err; echo "default rc=$?"
  for v in obsm3 obsm5; do
    FFTPIM_LIB=$V/libfftpim_$v.so timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_${v}_$rep.jsonl 2> $OUT/c4_${v}_$rep.err; echo "$v rc=$?"
  done
  FFTPIM_FFT_IP=1 timeout 900 python bench.py --no-cpu-baseline --steps 10 > $OUT/c4_fftip_$rep.jsonl 2> $OUT/c4_fftip_$rep.err; echo "fftip rc=$?"
done
python tools/showbench.py $OUT/c4_*.jsonl | grep -v fp64
