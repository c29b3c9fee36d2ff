"""Read-only bandwidth of the fold's access patterns (tm_probe_read_pattern) next to
a contiguous stream (tm_probe_read_bw), best of 5, GB/s.  Instrumentation."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_04863_b200 as tm  # noqa: E402

L = tm.lib()
L.tm_probe_read_pattern.restype = ctypes.c_int
L.tm_probe_read_pattern.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
buf = torch.ones(2 ** 31, dtype=torch.int8, device="cuda")
s = torch.cuda.current_stream()


def best(fn, nbytes, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return nbytes / (min(ts) * 1e-3) / 1e9


out = {"contiguous": best(lambda: tm.probe_read_bw(buf, stream=s), 2 ** 31)}
cases = [("cfg5 fold: ldx 64K, 4K pieces, R 896, groups fastest", 65536, 4096, 32768, 896, 0, 0),
         ("cfg5 fold, row chunks fastest", 65536, 4096, 32768, 896, 1, 0),
         ("ldx 64K, 8K pieces, R 896", 65536, 8192, 32768, 896, 0, 0),
         ("ldx 64K, 16K pieces, R 896", 65536, 16384, 32768, 896, 0, 0),
         ("ldx 64K, 32K pieces, R 896", 65536, 32768, 32768, 896, 0, 0),
         ("cfg4 fold: ldx 16K, 4K pieces, R 256", 16384, 4096, 2 ** 31 // 16384, 256, 0, 0),
         ("cfg4, R 1024", 16384, 4096, 2 ** 31 // 16384, 1024, 0, 0),
         ("cfg2-like: ldx 4K (contiguous 32K stages), R 256", 4096, 4096, 2 ** 31 // 4096, 256, 0, 0),
         ("cfg5 pattern, 296 CTAs", 65536, 4096, 32768, 896, 0, 296),
         ("cfg5 pattern, R 3584 (one item per CTA)", 65536, 4096, 32768, 3584, 0, 0)]
for name, ldx, w, rows, R, order, grid in cases:
    def fn(ldx=ldx, w=w, rows=rows, R=R, order=order, grid=grid):
        rc = L.tm_probe_read_pattern(buf.data_ptr(), ldx, w, rows, R, order, grid, s.cuda_stream)
        assert rc == 0, L.tm_last_error()
    out[name] = best(fn, ldx * rows)
print(json.dumps(out, indent=1))
