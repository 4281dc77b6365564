import sys, traceback
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import test_gpu_fuse_decode as T
import numpy as np
for case in [(136, 52, 96, 3, 2), (136, 52, 96, 1, 2), (64, 32, 128, 4, 1), (136, 52, 96, 3, 1)]:
    for fuse in (False, True):
        try:
            out, _ = T.run(*case, 5, fuse)
            print(case, fuse, "ok", float(np.abs(out[0]).sum()), flush=True)
        except Exception as e:
            print(case, fuse, "ERR", repr(e), flush=True)
