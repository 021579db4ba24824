"""Reader for the p2r checkpoint container.

The container is written and loaded by libp2r (csrc/engine/checkpoint.cpp);
this module only *reads* it on the host, so a checkpoint can be inspected
(manifest, StageState, any named buffer) without a GPU:

    m = read_manifest("pseudo.p2rckpt")
    m["stage"], m["config"]["d_model"], m["buffers"]["param/layer.0.attn.wq"]["shape"]
    w = read_buffer("pseudo.p2rckpt", "adam_m/layer.0.attn.wq")

Layout: magic "P2RCKPT\\0", u32 version (1), u32 manifest length, UTF-8
manifest, then little-endian fp32 buffers at 64-byte aligned offsets.
"""
import struct

import numpy as np

MAGIC = b"P2RCKPT\x00"
VERSION = 1


def read_manifest(path: str) -> dict:
    with open(path, "rb") as f:
        head = f.read(16)
        if len(head) != 16 or head[:8] != MAGIC:
            raise ValueError(f"checkpoint: not a p2r checkpoint: {path}")
        version, mlen = struct.unpack("<II", head[8:16])
        if version != VERSION:
            raise ValueError(f"checkpoint: unsupported format version {version}")
        text = f.read(mlen).decode("utf-8")
    out = {"version": version, "buffers": {}, "order": []}
    for line in text.splitlines():
        tok = line.split()
        if not tok:
            continue
        key = tok[0]
        if key == "config":
            kv = dict(zip(tok[1::2], tok[2::2]))
            cfg = {k: int(v) for k, v in kv.items() if k != "capacity_factor"}
            cfg["capacity_factor"] = float.fromhex(kv["capacity_factor"])
            out["config"] = cfg
        elif key == "ep":
            out["ep"] = (int(tok[1]), int(tok[2]))
        elif key == "stage":
            out["stage"] = tok[1]
        elif key in ("global_step", "samples_consumed", "rng_state", "last_eval_step"):
            out[key] = int(tok[1])
        elif key == "wall_time_s":
            out[key] = float.fromhex(tok[1])
        elif key == "adamw":
            out["adamw"] = {"attached": tok[1] == "1", "b1": float.fromhex(tok[2]), "b2": float.fromhex(tok[3]),
                            "eps": float.fromhex(tok[4]), "wd": float.fromhex(tok[5]), "step_count": int(tok[6])}
        elif key == "buffer":
            name, dtype, nd = tok[1], tok[2], int(tok[3])
            shape = tuple(int(x) for x in tok[4:4 + nd])
            out["buffers"][name] = {"dtype": dtype, "shape": shape, "offset": int(tok[4 + nd], 16),
                                    "bytes": int(tok[5 + nd], 16)}
            out["order"].append(name)
    return out


def read_buffer(path: str, name: str, manifest: dict = None) -> np.ndarray:
    m = manifest or read_manifest(path)
    e = m["buffers"][name]
    with open(path, "rb") as f:
        f.seek(e["offset"])
        raw = f.read(e["bytes"])
    if len(raw) != e["bytes"]:
        raise ValueError(f"checkpoint: truncated buffer {name}")
    return np.frombuffer(raw, dtype="<f4").reshape(e["shape"]).copy()
