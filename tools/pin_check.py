import sys
sys.path.insert(0, "/root/repo")
from paper_2601_19911_b200 import B200Device, _native
d = B200Device()
lib = _native.load()
a = _native.host_array(10_000_000)
print("arena array pinned:", lib.golp_host_is_pinned(_native.ptr(a)), hex(_native.ptr(a)), _native.last_error())
import numpy as np
b = np.empty(10_000_000, np.uint32)
print("numpy array pinned:", lib.golp_host_is_pinned(_native.ptr(b)))
