"""Host-side checkpoint reader (paper_2110_03888_b200/checkpoint.py) against a
container assembled here byte-by-byte from the format spec (
csrc/engine/checkpoint.cpp header). No GPU: documents and pins the layout."""
import struct

import numpy as np
import pytest

from paper_2110_03888_b200.checkpoint import MAGIC, read_buffer, read_manifest


def build(path, bufs, version=1, magic=MAGIC, n_experts=0, ep=(1, 0)):
    names = list(bufs)

    def manifest(offs):
        lines = ["p2r-checkpoint 1",
                 "config d_model 8 d_ff 32 n_layers_graph 2 n_layers_params 1 n_heads 2 vocab_size 260 "
                 f"seq_len 4 n_experts {n_experts} n_prototypes 1 n_shards {ep[0]} capacity_factor {float(1.25).hex()}",
                 f"ep {ep[0]} {ep[1]}", "stage PSEUDO", "global_step 3", "samples_consumed 96",
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


def moe_buffers(rng, experts):
    out = {}
    for kind in ("param", "adam_m", "adam_v"):
        out[f"{kind}/tok_emb"] = rng.standard_normal((260, 8)).astype(np.float32)
        out[f"{kind}/layer.0.moe.gate"] = rng.standard_normal((8, 4)).astype(np.float32)
        for e in experts:
            out[f"{kind}/layer.0.moe.expert.{e}.w1"] = rng.standard_normal((8, 32)).astype(np.float32)
            out[f"{kind}/layer.0.moe.expert.{e}.b2"] = rng.standard_normal(8).astype(np.float32)
    return out


def test_redistribute_checkpoints_host(tmp_path):
    """SPEC redistribute_experts across GPU counts: 1 -> 2 -> 4 -> 1 shards through the
    library's host-only re-shard; every buffer lands on its shard unchanged."""
    import paper_2110_03888_b200 as p2r
    rng = np.random.default_rng(3)
    full = moe_buffers(rng, range(4))
    src = str(tmp_path / "full.p2rckpt")
    build(src, full, n_experts=4)
    two = [str(tmp_path / f"two{r}.p2rckpt") for r in range(2)]
    p2r.redistribute_checkpoints([src], two)
    for r, path in enumerate(two):
        m = read_manifest(path)
        assert m["ep"] == (2, r) and m["config"]["n_shards"] == 2 and m["global_step"] == 3
        experts = sorted({int(n.split(".")[4]) for n in m["buffers"] if ".moe.expert." in n})
        assert experts == [2 * r, 2 * r + 1]
        for n in m["buffers"]:
            assert np.array_equal(read_buffer(path, n, m), full[n]), n
    four = [str(tmp_path / f"four{r}.p2rckpt") for r in range(4)]
    p2r.redistribute_checkpoints(two, four)
    back = str(tmp_path / "back.p2rckpt")
    p2r.redistribute_checkpoints(four, [back])
    m = read_manifest(back)
    assert m["ep"] == (1, 0) and set(m["buffers"]) == set(full)
    for n in full:
        assert np.array_equal(read_buffer(back, n, m), full[n]), n
    with pytest.raises(p2r.P2RInvalidArgument, match="divisible by new shard count"):
        p2r.redistribute_checkpoints([src], [str(tmp_path / f"x{r}") for r in range(3)])
    with pytest.raises(p2r.P2RInvalidArgument, match="is not shard"):
        p2r.redistribute_checkpoints([two[1], two[0]], [str(tmp_path / "y")])
