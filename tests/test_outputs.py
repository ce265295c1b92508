"""Run artifacts are byte-identical to the reference's writers
(outputs.py:3-105; fixtures from tests/golden/make_golden.py gen_outputs)."""

import numpy as np
import pytest
import torch

from paper_2503_05046_b200 import outputs as po


def test_frame_bytes_match_reference(golden, tmp_path):
    g = golden("outputs")
    assert po.frame_bytes(float(g["time"]), g["x"], g["v"]) == g["frame_v"].tobytes()
    assert po.frame_bytes(0.5, g["x"]) == g["frame_nov"].tobytes()
    po.write_frame(tmp_path / "a.bin", float(g["time"]), torch.as_tensor(g["x"]),
                   torch.as_tensor(g["v"]))
    assert (tmp_path / "a.bin").read_bytes() == g["frame_v"].tobytes()
    t, x, v = po.read_frame(tmp_path / "a.bin")
    assert t == float(g["time"]) and np.array_equal(x, g["x"]) and np.array_equal(v, g["v"])


def test_csv_frame_and_contact_log_match_reference(golden, tmp_path):
    g = golden("outputs")
    po.write_frame_csv(tmp_path / "c.csv", float(g["time"]), g["x"], g["v"])
    assert (tmp_path / "c.csv").read_bytes() == g["frame_csv"].tobytes()
    log = po.ContactLogWriter(tmp_path / "contacts.csv", ["ground", "pusher"])
    wr = g["wrench"]
    log.log_step(0.002, {"ground": wr[0], "pusher": wr[1]})
    log.log_step(0.004, {"ground": -wr[0], "pusher": 2 * wr[1]})
    log.close()
    assert (tmp_path / "contacts.csv").read_bytes() == g["contact_log"].tobytes()


def test_async_writer_host_tensors(golden, tmp_path):
    g = golden("outputs")
    w = po.AsyncFrameWriter(depth=2)
    for k in range(3):
        w.submit(tmp_path / f"f{k}.bin", float(g["time"]) if k == 0 else 0.5 * k,
                 torch.as_tensor(g["x"]), torch.as_tensor(g["v"]) if k == 0 else None)
    w.close()
    assert (tmp_path / "f0.bin").read_bytes() == g["frame_v"].tobytes()
    assert po.read_frame(tmp_path / "f2.bin")[0] == 1.0


def test_bad_magic_raises(tmp_path):
    (tmp_path / "x.bin").write_bytes(b"XXXX" + bytes(24))
    with pytest.raises(ValueError):
        po.read_frame(tmp_path / "x.bin")
