"""a1/a2 timing (CPU): JSONL trace parse + layer-summed activation matrix —
this library's host C++ loader vs the compiled reference (nlohmann), on a
SURVEY §8 a1-sized synthetic trace (written by the byte-identical writer)."""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.pyoracle import Reference, have_reference  # noqa: E402
from paper_2604_23150_b200 import trace as tr  # noqa: E402

E, k, L = 128, 8, 16
model = tr.ModelConfig("m", E, k, L)
spec = tr.SyntheticTraceSpec(4, 2048, 32, 0.6, 16.0, 1)
t = tr.generate_synthetic_trace(spec, model)
path = Path(tempfile.mkdtemp()) / "trace.jsonl"
t.write(path)
mb = path.stat().st_size / 1e6
import ctypes as C  # noqa: E402
from paper_2604_23150_b200 import _abi  # noqa: E402
h = C.c_void_p()
t0 = time.perf_counter()  # the C ABI call alone (file read + parse + validation)
_abi.call("mpb_trace_read_file", str(path).encode(), E, k, L, C.byref(h))
t1 = time.perf_counter()
_abi.lib().mpb_trace_destroy(h)
mine = tr.read_trace_file(path, model)  # + the Python mirror's array export
tm = time.perf_counter()
tr.build_activation_matrix_summed(mine, E, 1)
t2 = time.perf_counter()
out = {"records": len(mine), "mbytes": round(mb, 1), "threads": os.cpu_count(),
       "parse_s": round(t1 - t0, 3), "parse_mb_s": round(mb / (t1 - t0), 1),
       "matrix_s": round(t2 - tm, 3)}
if have_reference():
    rp, rm, rn = Reference().bench_parse(path, E, k, L)
    assert rn == len(mine)
    out.update(ref_parse_s=round(rp, 3), ref_parse_mb_s=round(mb / rp, 1), ref_matrix_s=round(rm, 3),
               parse_speedup=round(rp / (t1 - t0), 1))
print(json.dumps(out))
os.remove(path)
