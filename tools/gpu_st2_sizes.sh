# 2D stencil kernel choice: strip march vs tile kernel over grid sizes
mkdir -p gpurun_out
python -c "from paper_1703_01202_b200 import build as B; B.build()" || exit 1
for v in "strip:-DST2_STRIP_MIN=0" "tile:-DST2_STRIP_MIN=1000000000000L"; do
  name=${v%%:*}; flags=${v#*:}
  PFC_VARIANT_SOURCES=stencil2d.cu PFC_LIB_NAME=libpfc_$name.so PFC_EXTRA_NVCC_FLAGS="$flags" python -c "from paper_1703_01202_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || echo "build $name failed"
  echo "== $name"
  PFC_LIB_PATH=paper_1703_01202_b200/lib/libpfc_$name.so timeout 300 python tools/kernel_probe.py st2dsz 20 2>&1 | grep -E "(jv|residual) .*n=  20"
done
