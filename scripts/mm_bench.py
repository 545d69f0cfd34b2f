"""SURVEY 8(f)3 measurement: Matrix Market -> CSR ingestion, ours (parallel host
parse + device sort/dedup, hdcg_read_matrix_market) vs the reference's
io.cpp/coo.cpp (oracle/_ref), on a 7-point Laplacian written as a general
coordinate file.  Checks the two CSRs are identical; prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 128
path = sys.argv[2] if len(sys.argv) > 2 else f"/tmp/lap{g}.mtx"
rp, col, val = synth.laplacian7(g, g, g)
n = len(rp) - 1
nnz = int(rp[-1])
t0 = time.perf_counter()
rows = np.repeat(np.arange(1, n + 1), np.diff(rp))
perm = np.random.default_rng(0).permutation(nnz)  # entries in random order, like an unsorted export
with open(path, "w") as f:
    f.write(f"%%MatrixMarket matrix coordinate real general\n{n} {n} {nnz}\n")
    body = np.char.add(np.char.add(np.char.add(rows[perm].astype(str), " "),
                                   np.char.add((col[perm].astype(np.int64) + 1).astype(str), " ")),
                       np.char.add(val[perm].astype(int).astype(str), "\n"))
    f.write("".join(body.tolist()))
t_write = time.perf_counter() - t0
size = os.path.getsize(path)
H.init(0)
H.read_matrix_market(path).free()  # warm: page cache, CUDA context, pools
t0 = time.perf_counter()
d = H.read_matrix_market(path)
t_ours = time.perf_counter() - t0
got = H.csr_from_device(d)
out = {"what": "Matrix Market -> CSR", "file": f"7-pt Laplacian {g}^3, general coordinate, shuffled",
       "bytes": size, "nnz": nnz, "ours_s": round(t_ours, 4), "ours_mb_s": round(size / t_ours / 1e6, 1),
       "host_threads": os.cpu_count(), "write_s": round(t_write, 2)}
assert np.array_equal(got.row_ptr.astype(np.int64), rp.astype(np.int64))
assert np.array_equal(got.col_ind, col) and got.values.tobytes() == val.tobytes()
try:
    from oracle.oracle import Ref
    R = Ref()
    R.read_matrix_market(path)
    t0 = time.perf_counter()
    w = R.read_matrix_market(path)
    out["reference_s"] = round(time.perf_counter() - t0, 4)
    out["reference_mb_s"] = round(size / out["reference_s"] / 1e6, 1)
    out["speedup"] = round(out["reference_s"] / t_ours, 1)
    assert np.array_equal(np.asarray(w[0]), rp.astype(np.int64)) and np.array_equal(np.asarray(w[1]), col)
    out["identical_to_reference"] = True
except Exception as e:  # noqa: BLE001
    out["reference_error"] = repr(e)[:200]
print(json.dumps(out))
os.remove(path)
