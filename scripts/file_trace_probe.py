import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1403_7295_b200 import paes
O = oracle.Oracle(); key = O.sweep(3,16)
n=(4<<30)+7
src='/dev/shm/paes_tr_in.bin'; ct='/dev/shm/paes_tr_ct.bin'
buf=np.empty(n,dtype=np.uint8); O.counter_fill_into(3,0,n,buf.ctypes.data); buf.tofile(src); del buf
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
