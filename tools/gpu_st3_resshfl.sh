# 3D residual: left/right stage-1 neighbours of s by warp shuffles (ST3_RES_SHFL=1, new default)
# vs all eight from the s plane (=0); bitwise comparison of the two and parity vs the oracle
mkdir -p gpurun_out
export ST3_VARIANTS="splane:-DST3_RES_SHFL=0"
bash tools/gpu_st3_variants.sh > gpurun_out/st3_resshfl.log 2>&1
for n in "512 512 512" "96 64 40" "70 50 33"; do
  python tools/st3_res_cmp.py /tmp/res_a.pt $n >> gpurun_out/st3_resshfl.log 2>&1
  PFC_LIB_PATH=paper_1703_01202_b200/lib/libpfc_splane.so python tools/st3_res_cmp.py /tmp/res_b.pt $n >> gpurun_out/st3_resshfl.log 2>&1
  python -c "import torch; a=torch.load('/tmp/res_a.pt'); b=torch.load('/tmp/res_b.pt'); print('bitwise equal [$n]:', bool((a==b).all()), float((a-b).abs().max()))" >> gpurun_out/st3_resshfl.log 2>&1
done
python tools/st3_check.py 128 res >> gpurun_out/st3_resshfl.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "residual or stencil or operator or 3d" >> gpurun_out/st3_resshfl.log 2>&1
cat gpurun_out/st3_resshfl.log | tail -30
