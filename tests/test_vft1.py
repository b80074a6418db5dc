"""VFT1 I/O (paper_2604_12798_b200/vft1.py) against the reference's format
(src/tensor_io.py): fixtures written by the reference writer (tests/golden/make_vft1.py),
and the reference's own tests (tests/test_io.py) restated for this reader / writer."""

import os

import numpy as np
import pytest

from paper_2604_12798_b200 import vft1

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "vft1")


def test_reads_reference_files_exactly():
    m = np.load(os.path.join(FIX, "m.npy"))
    assert np.array_equal(vft1.read_matrix(os.path.join(FIX, "m_f64.vft")), m)
    assert np.array_equal(vft1.read_matrix(os.path.join(FIX, "m_f32.vft")), m.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("code,name", [(vft1.DTYPE_F64, "m_f64.vft"), (vft1.DTYPE_F32, "m_f32.vft")])
def test_writer_is_byte_identical_to_reference(tmp_path, code, name):
    m = np.load(os.path.join(FIX, "m.npy"))
    vft1.write_matrix(tmp_path / "x.vft", m, code)
    assert (tmp_path / "x.vft").read_bytes() == open(os.path.join(FIX, name), "rb").read()


def _corrupt(tmp_path, edit):
    path = tmp_path / "m.vft"
    vft1.write_matrix(path, np.ones((4, 4)))
    path.write_bytes(edit(bytearray(path.read_bytes())))
    return path


@pytest.mark.parametrize("edit,err", [
    (lambda b: bytes(b"X" + b[1:]), vft1.BadMagicError),
    (lambda b: bytes(b[:4] + bytes([9]) + b[5:]), vft1.BadDTypeError),
    (lambda b: bytes(b[:6] + bytes([1]) + b[7:]), vft1.HeaderError),
    (lambda b: bytes(b[:5] + bytes([3]) + b[6:]), vft1.HeaderError),
    (lambda b: bytes(b[:-3]), vft1.TruncatedError),
    (lambda b: bytes(b[:12]), vft1.TruncatedError),
    (lambda b: bytes(b[:6]), vft1.TruncatedError),
    (lambda b: bytes(b) + b"\x00", vft1.HeaderError),
])
def test_malformed_files(tmp_path, edit, err):
    # reference tests/test_io.py:33-78
    with pytest.raises(err):
        vft1.read_matrix(_corrupt(tmp_path, edit))


def test_write_rejects_non_2d_and_bad_dtype(tmp_path):
    with pytest.raises(vft1.HeaderError):
        vft1.write_matrix(tmp_path / "a.vft", np.zeros(4))
    with pytest.raises(vft1.BadDTypeError):
        vft1.write_matrix(tmp_path / "a.vft", np.zeros((2, 2)), 7)


def test_runner_errors_map_to_reference_exit_codes(tmp_path):
    from paper_2604_12798_b200 import runner
    with pytest.raises(runner.DataError) as e:
        runner.load_tensors(tmp_path)  # missing q.vft
    assert runner.exit_code(e.value) == 3
    with pytest.raises(runner.ConfigError) as e:
        runner._config(variant="naive")
    assert runner.exit_code(e.value) == 2
    assert runner.exit_code(vft1.TruncatedError("x")) == 3
    with pytest.raises(runner.ConfigError):
        runner._config(lam=2.0)
    q, k, v = runner.load_tensors(FIX)
    assert q.shape == (256, 64)
    with pytest.raises(runner.DataError):
        runner.problem_from(runner._config(q_block=128, k_block=96), q, k, v)  # 256 % 96 != 0
