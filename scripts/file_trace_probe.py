"""PAES_FILE_TRACE timeline of run_job on /dev/shm (4 GiB + 7): the Prealloc thread's run time and the writers'
total wait, with a replaced output reclaimed on a detached thread (1) or inside rename (0), and with no old
output at all (last two reps).  Developer probe; prints to stdout/stderr.

    python scripts/file_trace_probe.py
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1403_7295_b200 import paes
key = bytes(range(16))
n=(4<<30)+7
src='/dev/shm/paes_tr_in.bin'; ct='/dev/shm/paes_tr_ct.bin'
rng = np.random.default_rng(3)
with open(src, 'wb') as f:
    left = n
    while left:
        m = min(left, 256 << 20)
        f.write(rng.integers(0, 256, m, dtype=np.uint8).tobytes())
        left -= m
paes.encrypt_file(src,ct,key,workers=1)
os.environ['PAES_FILE_TRACE']='1'
for rec in ('1','0'):
    os.environ['PAES_FILE_ASYNC_RECLAIM']=rec
    for i in range(4):
        if rec=='0' and i>=2: os.unlink(ct)   # no old output at all
        r=paes.encrypt_file(src,ct,key,workers=1)
        print('reclaim',rec,'rep',i,'job',round(r['seconds'],4),flush=True)
        time.sleep(1.0)
os.unlink(src); os.unlink(ct)
