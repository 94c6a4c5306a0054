"""Compare attention harness dumps (O, dQKV as bf16) between variants: max |diff| / max |ref|."""
import sys
import numpy as np


def load(p):
    u = np.fromfile(p, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32)


ref = load(sys.argv[1])
for p in sys.argv[2:]:
    x = load(p)
    d = np.abs(x - ref)
    print(f'{{"cmp": "{p}", "max_abs": {d.max():.3e}, "ref_max": {np.abs(ref).max():.3e}, '
          f'"rel_l2": {np.linalg.norm(x - ref) / np.linalg.norm(ref):.3e}, "identical": {bool((x == ref).all())}}}')
