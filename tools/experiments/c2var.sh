mkdir -p gpurun_out/s33
V=paper_2312_02376_b200/lib/variants/libfftpim_k1t128.so
D=paper_2312_02376_b200/lib/libfftpim.so
for rep in 1 2; do
for lib in $D $V; do
 for fg in 0 1; do
  for cb in 222 296; do
   tag=$(basename $lib .so)_fg${fg}_cb${cb}_r$rep
   FFTPIM_LIB=$lib FFTPIM_FAR_GATE=$fg FFTPIM_CORR_BLOCKS=$cb python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s33/$tag.jsonl 2>&1
  done
 done
done
done
echo done
