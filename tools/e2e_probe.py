import time, ctypes, numpy as np, sys
sys.path.insert(0, '.')
import paper_1404_0774_b200 as fic
from paper_1404_0774_b200 import images
from paper_1404_0774_b200._lib import lib
from paper_1404_0774_b200.abi import MAPPING_DTYPE, FicStats, ptr
img = images.CONFIGS['cfg2'][0]()
p = fic.CodecParams(n=8, step=4)
for _ in range(5): fic.encode(img, p)
t = time.perf_counter()
for _ in range(50): fic.encode(img, p)
print('fic.encode', (time.perf_counter() - t) / 50 * 1e3, 'ms')
out = np.zeros(4096, MAPPING_DTYPE); st = FicStats(); L = lib()
t = time.perf_counter()
for _ in range(50): L.fic_encode(ptr(img), 512, 512, ctypes.byref(p.struct), ptr(out), ctypes.byref(st))
print('raw fic_encode', (time.perf_counter() - t) / 50 * 1e3, 'ms')
t = time.perf_counter()
for _ in range(50): np.zeros(4096, MAPPING_DTYPE)
print('np.zeros', (time.perf_counter() - t) / 50 * 1e3, 'ms')
