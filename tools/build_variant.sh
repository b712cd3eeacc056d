#!/usr/bin/env bash
# tools/build_variant.sh NAME "DEFS": corr_kernels.cu recompiled with DEFS, linked
# with the other objects into paper_2312_02376_b200/lib/variants/libfftpim_NAME.so
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2312_02376_b200/csrc
L=$R/paper_2312_02376_b200/lib
NCCL=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
mkdir -p $L/variants
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I$NCCL/include $2 -c $C/corr_kernels.cu -o $L/variants/corr_$1.o 2>/dev/null
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/variants/libfftpim_$1.so \
  $L/obj/fftpim.o $L/obj/build_kernels.o $L/obj/eval_kernels.o $L/obj/line_kernels.o $L/variants/corr_$1.o \
  $L/obj/fft_kernels.o $L/obj/sweep_kernels.o $L/obj/direct_kernels.o -L/usr/local/cuda/lib64 -lcufft -cudart static \
  -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=/usr/local/cuda/lib64 -Xlinker -rpath=$NCCL/lib
echo built $1
