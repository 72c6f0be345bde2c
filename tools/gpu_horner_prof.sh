# phase timers (-DCL2_PROF) of the TMEM subdomain kernel: direct 63-point stencil vs Horner-in-T
mkdir -p gpurun_out
L=gpurun_out/horner_prof.log; : > $L
for lib in libpfc_prof.so libpfc_hprof.so; do
  echo "== $lib" >> $L
  PFC_LIB_PATH=$PWD/paper_1703_01202_b200/lib/$lib timeout 600 python tools/cl2_phase_probe.py 512 >> $L 2>&1
done
cat $L
