cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 600 python tools/smem_default_probe.py st0 > gpurun_out/store_mode.jsonl 2>&1
for sm in 1 2; do
  touch paper_2602_04103_b200/csrc/sbcache.cu
  make -s all QR_EXTRA=-DQR_STORE_MODE=$sm >> gpurun_out/make.log 2>&1
  timeout 600 python tools/smem_default_probe.py st$sm >> gpurun_out/store_mode.jsonl 2>&1
done
