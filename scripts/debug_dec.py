import os, random, sys
sys.path.insert(0, os.getcwd())
from paper_1403_7295_b200 import paes
import oracle
O = oracle.Oracle()
rnd = random.Random(11)
bad = []
for n in list(range(0, 70)) + [255, 256, 257, 4095, 4096, 4097, 65535, 65536, 65537, 100001]:
    key = bytes(rnd.getrandbits(8) for _ in range(16))
    data = os.urandom(n)
    ct = paes.encrypt_bytes(data, key)
    assert ct == O.encrypt_chunk(data, True, key)
    pt = paes.decrypt_bytes(ct, key)
    ref = O.decrypt_chunk(ct, True, key)
    raw = paes.decrypt_chunk(ct, False, key)
    rawo = O.ecb(1, ct, key)
    if pt != data:
        diff = next((i for i in range(min(len(pt), len(data))) if pt[i] != data[i]), None)
        rd = next((i for i in range(len(raw)) if raw[i] != rawo[i]), None)
        bad.append((n, len(pt), len(data), diff, ref == data, rd, len(ct)))
print("bad", bad)
