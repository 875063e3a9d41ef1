#!/bin/bash
# A/B of the fused-stage FFT launch variants (QVA_FS_ROWV / QVA_FS_COLV index the per-length
# variant lists of kernels_fft_fs.cu): cfg3 and 12! per p=4 evolution.
for v in "$@"; do
  echo "== $v"; env $v python tools/time_qwoa.py 3 2>&1 | grep FFT
done
