"""Small driver for ncu: one launch each of the encrypt, decrypt, batch
encrypt and batch decrypt kernels on 1 GiB of device-generated data (plus
warm-up launches).

    python scripts/profile_kernels.py
    ncu --set full --clock-control none -k regex:"ecb_kernel|batch_kernel" -s 4 -c 4 -o prof python scripts/profile_kernels.py
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1403_7295_b200 import paes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 30)
rk = paes.round_keys(paes.sweep(3, 16))
a = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
b = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
paes.counter_fill_device(3, 0, n, a.data_ptr())
# batch layout: 1 GiB split into log-uniform messages like config 5
lens = paes.batch_lengths(4, 4096)
off, in_off, out_off, L2 = 0, [], [], []
for L in lens:
    if off + L + 16 > n:
        break
    in_off.append(off)
    out_off.append(off)
    L2.append(L)
    off += L + 16
rks = np.frombuffer(os.urandom(16 * len(L2)), dtype=np.uint8)
rk_all = b"".join(paes.round_keys(bytes(rks[16 * i:16 * i + 16])) for i in range(len(L2)))
plan = paes.BatchPlan(0, in_off, out_off, L2, rk_all, True)
dplan = paes.BatchPlan(1, out_off, in_off, [x + 16 for x in L2], rk_all, True)
# warm-up: one of each
paes.ecb_device(0, a.data_ptr(), b.data_ptr(), n, rk)
paes.ecb_device(1, b.data_ptr(), a.data_ptr(), n, rk)
plan.run(a.data_ptr(), b.data_ptr())
dplan.run(b.data_ptr(), a.data_ptr())
torch.cuda.synchronize()
# profiled: encrypt, decrypt, batch encrypt (x3 each when sizing a launch list)
for _ in range(3 if len(sys.argv) > 1 else 1):
    paes.ecb_device(0, a.data_ptr(), b.data_ptr(), n, rk)
    paes.ecb_device(1, b.data_ptr(), a.data_ptr(), n, rk)
    plan.run(a.data_ptr(), b.data_ptr())
    dplan.run(b.data_ptr(), a.data_ptr())
torch.cuda.synchronize()
print("ok", len(L2), "messages")
