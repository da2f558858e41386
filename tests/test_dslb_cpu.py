"""The DSLB lookup-batch file (table.hpp:235-305) on CPU: the host writer and
reader against the reference's own save_lookup_batch / load_lookup_batch
(oracle/_ref), and the error behaviour of every loader — the reference, the
Python host reader and the C-ABI's device loader (sp_ingest_batch_file
raises these before it touches a GPU) — on corrupted files."""
import json
import os
import struct

import numpy as np
import pytest

from oracle import lookup as orc
from oracle import ref
from paper_2210_02023_b200.api import (LookupBatch, ShardplanError, ingest_batch_file,
                                       load_lookup_batch, save_lookup_batch)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden():
    with open(os.path.join(GOLD, "ref_dslb.json")) as f:
        return json.load(f)


def test_golden_file_reads_back():
    g = _golden()
    b = load_lookup_batch(os.path.join(GOLD, "ref_batch.dslb"))
    assert (b.num_tables, b.batch_size) == (g["num_tables"], g["batch_size"])
    assert (len(b.offsets), len(b.indices)) == (g["offsets_len"], g["indices_len"])
    assert int(b.offsets.sum()) == g["offsets_sum"] and int(b.indices.sum()) == g["indices_sum"]
    off, idx, T, B = ref.load_lookup_batch(os.path.join(GOLD, "ref_batch.dslb"))
    np.testing.assert_array_equal(b.offsets, off)
    np.testing.assert_array_equal(b.indices, idx)


@pytest.mark.parametrize("T,B,seed", [(6, 64, 1), (3, 5, 2), (0, 4, 3), (2, 3, -1)])
def test_writer_is_byte_identical_to_reference(tmp_path, T, B, seed):
    if seed < 0:  # no lookups at all
        off, idx = np.zeros(T * B + 1, dtype=np.int64), np.zeros(0, dtype=np.int64)
    else:
        tables = [{"id": t, "dim": 16, "hash_size": 100 + 50 * t, "pooling_factor": 2.0 + t,
                   "table_size_gb": 1e-5, "dist": [1.0] + [0.0] * 16} for t in range(T)]
        off, idx = (orc.synth_batch(tables, B, seed) if T else
                    (np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int64)))
    ours, theirs = tmp_path / "ours.dslb", tmp_path / "ref.dslb"
    save_lookup_batch(LookupBatch(idx, off, T, B), str(ours))
    ref.save_lookup_batch(str(theirs), off, idx, T, B)
    assert ours.read_bytes() == theirs.read_bytes()
    back = load_lookup_batch(str(theirs))
    np.testing.assert_array_equal(back.offsets, off)
    np.testing.assert_array_equal(back.indices, idx)


def _file(offsets, indices, T, B, version=1, magic=b"DSLB", offsets_len=None, cut=None):
    raw = (magic + struct.pack("<IIIQ", version, T, B,
                               len(offsets) if offsets_len is None else offsets_len)
           + np.asarray(offsets, "<i8").tobytes() + struct.pack("<Q", len(indices))
           + np.asarray(indices, "<i8").tobytes())
    return raw if cut is None else raw[:cut]


OFF = [0, 2, 3, 3, 5]  # T = 2, B = 2
IDX = [4, 1, 0, 2, 3]
CASES = {
    "valid": _file(OFF, IDX, 2, 2),
    "empty_file": b"",
    "short_magic": b"DSL",
    "bad_magic": _file(OFF, IDX, 2, 2, magic=b"DSLX"),
    "version_2": _file(OFF, IDX, 2, 2, version=2),
    "cut_in_header": _file(OFF, IDX, 2, 2, cut=14),
    "cut_in_offsets": _file(OFF, IDX, 2, 2, cut=24 + 8 * 3),
    "cut_in_indices_len": _file(OFF, IDX, 2, 2, cut=24 + 8 * 5 + 4),
    "cut_in_indices": _file(OFF, IDX, 2, 2, cut=24 + 8 * 5 + 8 + 8 * 4),
    "huge_offsets_len": _file(OFF, IDX, 2, 2, offsets_len=1 << 40),
    "offsets_len_mismatch": _file(OFF + [5], IDX, 2, 2),
    "zero_batch": _file([0], [], 2, 0),
    "negative_tables": _file([0], [], 0xFFFFFFFF, 2),
    "offsets_not_at_zero": _file([1, 2, 3, 3, 5], IDX, 2, 2),
    "offsets_decrease": _file([0, 3, 2, 3, 5], IDX, 2, 2),
    "last_offset_mismatch": _file([0, 2, 3, 3, 4], IDX, 2, 2),
    "trailing_bytes": _file(OFF, IDX, 2, 2) + b"\x00" * 7,
}


def _ref_status(path):
    try:
        ref.load_lookup_batch(path)
        return 0
    except ref.RefError as e:
        return e.code


def _status(fn):
    try:
        fn()
        return 0
    except ShardplanError as e:
        return e.status


@pytest.mark.parametrize("name", sorted(CASES))
def test_corrupted_files_fail_like_the_reference(tmp_path, name):
    path = str(tmp_path / f"{name}.dslb")
    with open(path, "wb") as f:
        f.write(CASES[name])
    want = _ref_status(path)
    assert (want == 0) == (name in ("valid", "trailing_bytes")), (name, want)
    assert _status(lambda: load_lookup_batch(path)) == want, name
    if want != 0:
        # the device loader rejects it on the host, before any CUDA call
        assert _status(lambda: ingest_batch_file(path, [16, 16], [10, 10])) == want, name


def test_missing_file_and_dims_mismatch(tmp_path):
    missing = str(tmp_path / "nope.dslb")
    assert _status(lambda: ingest_batch_file(missing, [16], [10])) == _ref_status(missing) == 10
    path = str(tmp_path / "ok.dslb")
    with open(path, "wb") as f:
        f.write(CASES["valid"])
    e = _status(lambda: ingest_batch_file(path, [16, 16, 16], [10, 10, 10]))
    assert e == 10  # "dims/hash_sizes length != num_tables" (bad_input)
