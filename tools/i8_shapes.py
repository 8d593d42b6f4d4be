"""int8 tcgen05.mma throughput vs N (M=128, K=32, back to back): A from shared
memory (SS) or from tensor memory (TS), B from shared memory."""
import sys
sys.path.insert(0, '.')
from paper_1708_01135_b200 import _lib
h = _lib.Handle(0)
for n in (16, 32, 48, 64, 80, 96, 128, 192, 256):
    print(f"N={n:3d}  SS {h.probe_i8_shape(n):8.1f}  TS {h.probe_i8_shape_ts(n):8.1f} TOP/s",
          flush=True)
