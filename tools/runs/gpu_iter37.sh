cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 600 python tools/fm_c5_probe.py mb4 > gpurun_out/fm_minb.jsonl 2>&1
for mb in 5 6; do
  touch paper_2602_04103_b200/csrc/fm.cu
  make -s all QR_EXTRA=-DQR_FM_MINB=$mb >> gpurun_out/make.log 2>&1
  timeout 600 python tools/fm_c5_probe.py mb$mb >> gpurun_out/fm_minb.jsonl 2>&1
done
