# two-stage hybrid (libpfc_hy2.so, -DCL2T_HORNER=2): apply times, difference vs the direct form, 3D parity tests
mkdir -p gpurun_out
L=gpurun_out/horner3.log; : > $L
for lib in libpfc_hy2.so; do
  echo "== $lib" >> $L
  PFC_LIB_PATH=paper_1703_01202_b200/lib/$lib RAS3_VARIANTS=cl2p:3,cl2t:3 timeout 600 python tools/ras3_probe.py 512 3 >> $L 2>&1
  PFC_LIB_PATH=paper_1703_01202_b200/lib/$lib RAS3_VARIANTS=cl2p:3,cl2t:3 timeout 600 python tools/ras3_probe.py 128 10 >> $L 2>&1
done
cat $L
PFC_LIB_PATH=$PWD/paper_1703_01202_b200/lib/libpfc_hy2.so timeout 1200 python -m pytest tests -m gpu -x -q -k "3d or cfg4 or cfg5 or testD or 3D or ras" >> $L 2>&1; echo "tests rc=$?" >> $L
tail -4 $L
