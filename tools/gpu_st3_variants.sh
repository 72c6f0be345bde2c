# Timing-only diagnostic variants of the 3D stencil (only stencil3d.cu is rebuilt per variant)
mkdir -p gpurun_out
python -c "from paper_1703_01202_b200 import build as B; B.build()" || exit 1
for v in "base:" ${ST3_VARIANTS}; do
  name=${v%%:*}; flags=$(echo ${v#*:} | tr ',' ' ')
  if [ "$name" != base ]; then
    PFC_VARIANT_SOURCES=stencil3d.cu PFC_LIB_NAME=libpfc_$name.so PFC_EXTRA_NVCC_FLAGS="$flags" python -c "from paper_1703_01202_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || { echo "build $name failed"; continue; }
    lib=paper_1703_01202_b200/lib/libpfc_$name.so
  else
    lib=paper_1703_01202_b200/lib/libpfc.so
  fi
  echo "== $name"
  PFC_LIB_PATH=$lib timeout 300 python tools/kernel_probe.py jv3d 20 2>&1 | grep "jv .*n=  20"
  PFC_LIB_PATH=$lib timeout 300 python tools/kernel_probe.py res3d 20 2>&1 | grep "residual .*n=  20"
done
