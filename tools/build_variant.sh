#!/usr/bin/env bash
# tools/build_variant.sh NAME "DEFS" [SRC]: SRC.cu (default corr_kernels) recompiled with DEFS,
# linked with the other objects into paper_2312_02376_b200/lib/variants/libfftpim_NAME.so
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2312_02376_b200/csrc
L=$R/paper_2312_02376_b200/lib
SRC=${3:-corr_kernels}
NCCL=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
mkdir -p $L/variants
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I$NCCL/include $2 -c $C/$SRC.cu -o $L/variants/${SRC}_$1.o 2>/dev/null
OBJS=""
for f in fftpim build_kernels eval_kernels line_kernels corr_kernels fft_kernels sweep_kernels direct_kernels; do
  if [ "$f" = "$SRC" ]; then OBJS="$OBJS $L/variants/${SRC}_$1.o"; else OBJS="$OBJS $L/obj/$f.o"; fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/variants/libfftpim_$1.so $OBJS \
  -L/usr/local/cuda/lib64 -lcufft -cudart static \
  -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=/usr/local/cuda/lib64 -Xlinker -rpath=$NCCL/lib
echo built $1
