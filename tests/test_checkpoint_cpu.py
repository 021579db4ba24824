"""Host-side checkpoint reader (paper_2110_03888_b200/checkpoint.py) against a
container assembled here byte-by-byte from the format spec (
csrc/engine/checkpoint.cpp header). No GPU: documents and pins the layout."""
import struct

import numpy as np
import pytest

from paper_2110_03888_b200.checkpoint import MAGIC, read_buffer, read_manifest


def build(path, bufs, version=1, magic=MAGIC):
    names = list(bufs)

    def manifest(offs):
        lines = ["p2r-checkpoint 1",
                 "config d_model 8 d_ff 32 n_layers_graph 2 n_layers_params 1 n_heads 2 vocab_size 260 "
                 f"seq_len 4 n_experts 0 n_prototypes 1 n_shards 1 capacity_factor {float(1.25).hex()}",
                 "ep 1 0", "stage PSEUDO", "global_step 3", "samples_consumed 96",
                 f"wall_time_s {float(2.5).hex()}", "rng_state 11", "last_eval_step -1",
                 f"adamw 1 {float(np.float32(0.9)).hex()} {float(np.float32(0.999)).hex()} "
                 f"{float(np.float32(1e-8)).hex()} {float(np.float32(0.01)).hex()} 3",
                 f"buffers {len(names)}"]
        for n, o in zip(names, offs):
            a = bufs[n]
            lines.append(f"buffer {n} f32 {a.ndim} " + " ".join(str(d) for d in a.shape) +
                         f" {o:016x} {a.nbytes:016x}")
        return ("\n".join(lines) + "\nend\n").encode()

    text = manifest([0] * len(names))
    off, offs = -(-(16 + len(text)) // 64) * 64, []
    for n in names:
        offs.append(off)
        off = -(-(off + bufs[n].nbytes) // 64) * 64
    text = manifest(offs)
    with open(path, "wb") as f:
        f.write(magic + struct.pack("<II", version, len(text)) + text)
        for n, o in zip(names, offs):
            f.write(b"\0" * (o - f.tell()))
            f.write(bufs[n].astype("<f4").tobytes())


def test_reader_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    bufs = {"param/tok_emb": rng.standard_normal((260, 8)).astype(np.float32),
            "param/layer.0.attn.wq": rng.standard_normal((8, 8)).astype(np.float32),
            "adam_m/layer.0.ln1.g": rng.standard_normal(8).astype(np.float32)}
    path = str(tmp_path / "x.p2rckpt")
    build(path, bufs)
    m = read_manifest(path)
    assert m["stage"] == "PSEUDO" and m["global_step"] == 3 and m["wall_time_s"] == 2.5
    assert m["config"]["capacity_factor"] == 1.25 and m["config"]["n_layers_graph"] == 2
    assert m["adamw"]["attached"] and m["adamw"]["step_count"] == 3 and m["ep"] == (1, 0)
    assert m["order"] == list(bufs)
    for n, a in bufs.items():
        assert m["buffers"][n]["offset"] % 64 == 0
        assert np.array_equal(read_buffer(path, n, m), a)


def test_reader_rejects_bad_files(tmp_path):
    bufs = {"param/x": np.ones(4, np.float32)}
    bad = str(tmp_path / "bad.p2rckpt")
    build(bad, bufs, magic=b"NOTACKPT")
    with pytest.raises(ValueError, match="not a p2r checkpoint"):
        read_manifest(bad)
    v2 = str(tmp_path / "v2.p2rckpt")
    build(v2, bufs, version=2)
    with pytest.raises(ValueError, match="unsupported format version 2"):
        read_manifest(v2)
