"""DDM1 container -> device (dg_create_from_ddm), SURVEY 8(f)-2.  Files are written by the
reference's own ddm::write_ddm (oracle/_ref); the header / size error contract is compared with
the reference's ddm::read_ddm on the same corrupted files (CPU: these checks precede any device
work), and the streamed upload is checked for dose parity on the GPU."""
import os

import numpy as np
import pytest

import paper_2103_09683_b200 as dg
from oracle.oracle import liver_desk, prostate_desk


def _status(path):
    try:
        dg.DoseEngine.from_ddm(path)
        return 0
    except dg.Error as e:
        return e.status


@pytest.fixture(scope="module")
def ddm_file(ref, tmp_path_factory):
    m = ref.generate(liver_desk())
    p = str(tmp_path_factory.mktemp("ddm") / "liver.ddm")
    ref.write_ddm(m, p)
    return p, m


def _corrupt(src, dst, fn):
    b = bytearray(open(src, "rb").read())
    b = fn(b)
    open(dst, "wb").write(bytes(b))
    return dst


@pytest.mark.parametrize("case", ["magic", "version", "precision", "index", "reserved",
                                  "truncated_header", "truncated_values", "trailing", "empty"])
def test_header_and_size_errors_match_reference(ref, ddm_file, tmp_path, case):
    src, _ = ddm_file
    edits = {
        "magic": lambda b: b"DDM2" + b[4:],
        "version": lambda b: b[:4] + bytes([2]) + b[5:],
        "precision": lambda b: b[:5] + bytes([3]) + b[6:],
        "index": lambda b: b[:6] + bytes([3]) + b[7:],
        "reserved": lambda b: b[:7] + bytes([1]) + b[8:],
        "truncated_header": lambda b: b[:20],
        "truncated_values": lambda b: b[:-3],
        "trailing": lambda b: b + b"\0",
        "empty": lambda b: b"",
    }
    p = _corrupt(src, str(tmp_path / f"{case}.ddm"), edits[case])
    want = ref.read_ddm_status(p)
    assert want != 0
    assert _status(p) == want, (case, dg.Errc(want - 1).name)


def test_missing_file_is_io_failure(tmp_path):
    assert _status(str(tmp_path / "nope.ddm")) == 1 + dg.Errc.IoFailure


@pytest.mark.gpu
@pytest.mark.parametrize("gen", [liver_desk, prostate_desk])
def test_ddm_upload_dose_matches_reference(ref, port, tmp_path, gen):
    m = ref.generate(gen())
    p = str(tmp_path / "m.ddm")
    ref.write_ddm(m, p)
    x = port.seeded_vector(m.cols, 42)
    with dg.DoseEngine.from_ddm(p) as e:
        y = e.dose(x)
        back = e.copy_rows(0, m.rows)
    assert np.array_equal(back.col_indices, m.col) and np.array_equal(back.values, m.values)
    want = ref.spmv_rowchunk(m, x, 32, 4)
    assert np.array_equal(y.view(np.uint64), want.view(np.uint64))


@pytest.mark.gpu
def test_ddm_upload_invalid_matrix_is_validation_failure(ref, tmp_path):
    m = ref.generate(liver_desk())
    p = str(tmp_path / "bad.ddm")
    ref.write_ddm(m, p)
    b = bytearray(open(p, "rb").read())
    # first column index of a non-empty row -> out of range (cols = 6800 fits u16)
    col_off = 32 + 8 * (m.rows + 1)
    r = int(np.nonzero(np.diff(m.row_ptr.astype(np.int64)))[0][0])
    j = int(m.row_ptr[r])
    b[col_off + 2 * j: col_off + 2 * j + 2] = (65000).to_bytes(2, "little")
    open(p, "wb").write(bytes(b))
    assert ref.read_ddm_status(p) == 1 + dg.Errc.ValidationFailure
    assert _status(p) == 1 + dg.Errc.ValidationFailure


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [2, 5])
def test_ddm_row_shards_read_only_their_ranges(ref, port, tmp_path, parts):
    """A rank reads only its rows' byte ranges of the column and value sections (the layout is
    fixed by the header, io.cpp:67-96): each shard's handle holds its shard only, reports its
    place in the source matrix, and its d is bit-identical to the reference's rowchunk on the
    file's matrix (read by ddm::read_ddm's writer counterpart) for those rows."""
    m = ref.generate(prostate_desk())
    p = str(tmp_path / "m.ddm")
    ref.write_ddm(m, p)
    x = port.seeded_vector(m.cols, 42)
    want = ref.spmv_rowchunk(m, x, 32, 4)
    b = dg.partition_rows(m.row_ptr, parts)
    got = np.empty(m.rows)
    for g in range(parts):
        r0, r1 = int(b[g]), int(b[g + 1])
        with dg.DoseEngine.from_ddm(p, row_begin=r0, row_end=r1) as e:
            assert (e.info["row_begin"], e.info["row_end"], e.info["rows"]) == (r0, r1, r1 - r0)
            assert e.info["nnz"] == int(m.row_ptr[r1] - m.row_ptr[r0])
            assert e.info["read_ns"] > 0  # the reader's own time (sections -> device)
            # resident bytes are the shard's, not the file's
            assert e.info["device_bytes"] < 1.5 * (e.info["nnz"] * 4 + 8 * (r1 - r0)) + (8 << 20)
            got[r0:r1] = e.dose(x)
            back = e.copy_rows(0, r1 - r0)
            s0, s1 = int(m.row_ptr[r0]), int(m.row_ptr[r1])
            assert np.array_equal(back.col_indices, m.col[s0:s1])
            assert np.array_equal(back.values, m.values[s0:s1])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    with pytest.raises(dg.Error) as e:
        dg.DoseEngine.from_ddm(p, row_begin=5, row_end=m.rows + 1)
    assert e.value.code == dg.Errc.InvalidConfig
