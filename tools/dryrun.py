import sys, json, ctypes as C, numpy as np
sys.path.insert(0, ".")
from paper_1808_01364_b200 import _lib, GridSpec, generate_field, assemble_operator
dim, n, m, keep = (int(a) for a in sys.argv[1:5])
spec = GridSpec(dim, n, m)
A = assemble_operator(generate_field(spec, 1))
rp = np.ascontiguousarray(A.csr.indptr, np.int64); ci = np.ascontiguousarray(A.csr.indices, np.int32)
L = _lib.lib()
k = L.phif_plan_dryrun(dim, n, m, _lib.ptr(rp), _lib.ptr(ci), keep, None, 0)
buf = C.create_string_buffer(k + 1)
L.phif_plan_dryrun(dim, n, m, _lib.ptr(rp), _lib.ptr(ci), keep, buf, k + 1)
for lv in json.loads(buf.value.decode()): print(lv)
