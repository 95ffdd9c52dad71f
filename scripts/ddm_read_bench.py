"""DDM1 reader throughput: the reference's ddm::read_ddm (element-by-element get_uint_le loop,
io.cpp:132-159) vs dg_create_from_ddm (large preads into pinned buffers streamed to the device),
on the C1 matrix written by the reference's own writer.  The file is in the page cache for
both (just written): this compares the parse / copy paths, not the disk.

    python scripts/ddm_read_bench.py [out.json]

`read_s` is the reader alone (dg_info.read_ns: row_ptr read + checked, column / value sections
preaded and streamed to the device); `create_from_ddm_s` is the whole create (plus validation,
plan, slice build), next to `create_from_csr_s` for the same matrix from host arrays."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_09683_b200 as dg  # noqa: E402
from oracle.oracle import Oracle, c1_profile  # noqa: E402


def main():
    ref = Oracle("reference")
    m = ref.generate(c1_profile())
    path = os.path.join(tempfile.mkdtemp(), "c1.ddm")
    ref.write_ddm(m, path)
    size = os.path.getsize(path)
    out = {"file_bytes": size, "nnz": int(m.nnz), "rows": int(m.rows), "note": "page-cached file"}
    t0 = time.perf_counter()
    st = ref.read_ddm_status(path)
    out["reference_read_ddm_s"] = time.perf_counter() - t0
    assert st == 0, st
    for k in range(2):  # first create also loads the library / context
        t0 = time.perf_counter()
        with dg.DoseEngine.from_ddm(path, device=0) as e:
            dt = time.perf_counter() - t0
            assert e.info["nnz"] == m.nnz
            out["read_s"] = e.info["read_ns"] * 1e-9  # sections -> device, inside the create
        out["create_from_ddm_s"] = dt
        csr = dg.CsrMatrix(m.rows, m.cols, m.index_width, m.row_ptr, m.col, m.values, m.precision)
        t0 = time.perf_counter()
        with dg.DoseEngine.from_csr(csr, device=0) as e:
            out["create_from_csr_s"] = time.perf_counter() - t0
    out["reference_MBps"] = size / out["reference_read_ddm_s"] / 1e6
    out["create_from_ddm_MBps"] = size / out["create_from_ddm_s"] / 1e6
    out["read_MBps"] = size / out["read_s"] / 1e6
    out["read_vs_reference"] = out["read_MBps"] / out["reference_MBps"]
    line = json.dumps(out)
    print(line)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(line + "\n")


if __name__ == "__main__":
    main()
