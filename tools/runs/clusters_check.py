import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, gen, paper_2602_04103_b200 as qr
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device="cuda"); gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n)
p = torch.cuda.get_device_properties(0)
print("clusters", qr.qr_super_cache_clusters(h), "sms", p.multi_processor_count, "name", p.name)
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=serial,uuid,clocks.max.mem,clocks.mem", "--format=csv"], capture_output=True, text=True).stdout)
