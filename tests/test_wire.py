"""The store wire protocol (reference wire.py) against the reference's own
frames and a served-session transcript (tests/golden/wire.json, made by
tests/golden/make_golden.py gen_wire), plus a socket session against the
B200 store (reference tests/test_wire.py)."""

from __future__ import annotations

import io
import socket
import threading

import numpy as np
import pytest

from conftest import golden
from paper_2202_12429_b200 import wire as W
from paper_2202_12429_b200.errors import WireFormatError
from paper_2202_12429_b200.traces import EmbeddingKey, Schema

G = golden("wire.json")
KEYS = [EmbeddingKey(t, r) for t, r in G["keys"]]
VALS = np.asarray(G["values"], dtype=np.uint32).view(np.float32)


def test_frames_match_reference():
    assert W.encode_fetch(KEYS).hex() == G["fetch"]
    assert W.encode_fetch_resp(VALS).hex() == G["fetch_resp"]
    assert W.encode_write(KEYS, VALS).hex() == G["write"]
    assert W.encode_ack(7).hex() == G["ack"]


def test_codec_round_trips_and_errors():
    t, p = W.read_message(io.BytesIO(bytes.fromhex(G["write"])))
    assert t == W.MSG_WRITE
    keys, vals = W.decode_write(p)
    assert keys == KEYS and np.array_equal(vals, VALS)
    t, p = W.read_message(io.BytesIO(bytes.fromhex(G["fetch"])))
    assert t == W.MSG_FETCH and W.decode_fetch(p) == KEYS
    assert W.decode_ack(W.read_message(io.BytesIO(bytes.fromhex(G["ack"])))[1]) == 7
    assert W.read_message(io.BytesIO(b"")) is None
    with pytest.raises(WireFormatError):
        W.read_message(io.BytesIO(b"\x01\x00"))
    bad = bytearray(bytes.fromhex(G["ack"]))
    bad[5] = 9  # version
    with pytest.raises(WireFormatError):
        W.read_message(io.BytesIO(bytes(bad)))
    with pytest.raises(WireFormatError):
        W.encode_write(KEYS[:2], VALS)


@pytest.mark.gpu
def test_served_session_matches_reference():
    from paper_2202_12429_b200.store import ShardedStore

    s = G["session"]
    nt, rows, nd, dim = s["schema"]
    store = ShardedStore(Schema(nt, tuple(rows), nd, dim), s["num_shards"], s["seed"])
    out = io.BytesIO()
    assert W.serve_connection(store, io.BytesIO(bytes.fromhex(s["requests"])), out) == s["served"]
    assert out.getvalue().hex() == s["responses"]


@pytest.mark.gpu
def test_socket_session():
    from paper_2202_12429_b200.store import ShardedStore

    store = ShardedStore(Schema(1, (64,), 0, 3), 2, 5)
    a, b = socket.socketpair()
    t = threading.Thread(target=lambda: W.serve_connection(store, a.makefile("rb"), a.makefile("wb")))
    t.start()
    rf, wf = b.makefile("rb"), b.makefile("wb")
    keys = [EmbeddingKey(0, r) for r in (3, 9, 17)]
    before = W.remote_fetch(rf, wf, keys)
    np.testing.assert_array_equal(before, store.fetch(keys))
    vals = np.arange(9, dtype=np.float32).reshape(3, 3)
    assert W.remote_write(rf, wf, keys, vals) == 3
    np.testing.assert_array_equal(W.remote_fetch(rf, wf, keys), vals)
    wf.close()
    b.shutdown(socket.SHUT_WR)
    t.join(timeout=30)
    a.close()
    b.close()
