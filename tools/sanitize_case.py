"""Small extraction cases for compute-sanitizer (both paths, ragged sizes, tail word)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_04130_b200 as q
import qrng_synth as S

q.load_library()
for path in (q.PATH_GEMM, q.PATH_NTT):
    q.set_debug_path(path)
    for n, m, B in [(1024, 716, 37), (8192, 5734, 5), (256, 13, 3), (65536, 45875, 2)]:
        if path == q.PATH_GEMM and n % 128:
            continue
        raw = torch.from_numpy(S.random_bytes(n + m, B * n // 8)).cuda()
        seed = torch.from_numpy(S.random_bytes(n + m, (n + m - 1 + 7) // 8, tag=2)).cuda()
        out = q.toeplitz_extract(raw, B, n, m, seed)
        torch.cuda.synchronize()
q.set_debug_path(q.PATH_AUTO)
x = torch.from_numpy(S.adc_samples(1, 100_000)).cuda()
q.minentropy(x, 8, 1024, 0)
host = np.zeros(q.out_bytes(40, 716), np.uint8)
q.toeplitz_extract_host(S.random_bytes(3, 40 * 128), 40, 1024, 716, S.random_bytes(3, 218, tag=2), host)
print("sanitize case done")
