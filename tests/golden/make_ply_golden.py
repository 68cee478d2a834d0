"""Freeze PLY golden bytes by running the UNMODIFIED reference `fgbd.ply`.

Run in the build container only (the reference tree is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_ply_golden.py

Writes tests/golden/ply.npz + ply_index.json:
* `save/<case>`: reference `save_ply` bytes for clouds rebuilt from seeds
  (binary + ascii, quantized + float, colours on the .5 rounding edges);
* `load/<case>`: hand-built PLY files (mixed property types, skipped
  elements, unknown properties) with the cloud the reference parses;
* `errors`: malformed inputs with the exception class and message;
* `denoise/<case>`: `save_ply(denoise(load_ply(bytes)))` -- the fused
  `denoise_ply` target.
"""

from __future__ import annotations

import json
import os
import struct
import sys
import warnings
from pathlib import Path

sys.dont_write_bytecode = True
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import fgbd  # noqa: E402  (the reference)

OUT = Path(__file__).resolve().parent


def edge_colors(n, seed):
    """Colours on and around the half-up rounding edges plus the clamp ends."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 256, size=(n, 3)).astype(np.float64)
    frac = rng.choice(np.array([0.0, 0.5, 0.49999999999, 0.5000000001, 0.25, 0.75]),
                      size=(n, 3))
    c = np.clip(base + frac, 0, 255)
    c[:4] = [[0, 0.5, 255], [254.5, 255, 0.4999], [1.5, 2.5, 3.5], [0, 0, 0]]
    return c


def synth_cases():
    """(name, builder kwargs, cloud) for save/denoise fixtures."""
    out = []
    clean, _ = fgbd.generate_cloud("two-tone", 3000, bits=9, seed=3)
    noisy = fgbd.add_gaussian_noise(clean, 20.0, seed=4)
    out.append(("twotone3k", dict(kind="two-tone", n=3000, bits=9, seed=3, sigma=20.0,
                                  noise_seed=4), noisy))
    clean, _ = fgbd.generate_cloud("ramp", 1200, bits=7, seed=5)
    noisy = fgbd.add_gaussian_noise(clean, 10.0, seed=6)
    out.append(("ramp1200", dict(kind="ramp", n=1200, bits=7, seed=5, sigma=10.0,
                                 noise_seed=6), noisy))
    return out


def float_cloud(n, seed):
    rng = np.random.default_rng(seed)
    coords = rng.normal(size=(n, 3)) * np.array([1.0, 1e3, 1e-3])
    coords[0] = [0.1, -0.0, 1e30]
    return fgbd.PointCloud(coords, edge_colors(n, seed + 1), None)


def quant_edge_cloud(n, seed):
    rng = np.random.default_rng(seed)
    coords = rng.integers(0, 1 << 21, size=(n, 3))
    coords[0] = [0, 0, (1 << 21) - 1]
    return fgbd.PointCloud(coords, edge_colors(n, seed + 1), 21)


def header(fmt, elements):
    lines = ["ply", f"format {fmt} 1.0", "comment made by make_ply_golden"]
    for name, count, props in elements:
        lines.append(f"element {name} {count}")
        lines += [f"property {t} {p}" for p, t in props]
    lines.append("end_header")
    return ("\n".join(lines) + "\n").encode()


_FMT = {"char": "b", "uchar": "B", "short": "h", "ushort": "H", "int": "i", "uint": "I",
        "float": "f", "double": "d", "int8": "b", "uint8": "B", "int16": "h",
        "uint16": "H", "int32": "i", "uint32": "I", "float32": "f", "float64": "d"}


def binary_file(elements, rows_per_element, pre=b""):
    body = b""
    for (name, count, props), rows in zip(elements, rows_per_element):
        fmt = "<" + "".join(_FMT[t] for _, t in props)
        body += b"".join(struct.pack(fmt, *r) for r in rows)
    return header("binary_little_endian", elements) + body + pre


def load_cases():
    rng = np.random.default_rng(11)
    cases = {}
    # mixed integer types + an unknown double property + a skipped element first
    n = 257
    vprops = [("x", "short"), ("nx", "double"), ("y", "ushort"), ("z", "int"),
              ("red", "uchar"), ("green", "uint8"), ("alpha", "uchar"), ("blue", "uchar")]
    rows = [(int(rng.integers(0, 3000)), float(rng.normal()), int(rng.integers(0, 60000)),
             int(rng.integers(0, 1 << 20)), *[int(v) for v in rng.integers(0, 256, 4)])
            for _ in range(n)]
    cam = [("cx", "float"), ("cy", "float"), ("id", "int")]
    cam_rows = [(1.0, 2.0, 7), (3.5, -1.0, 9)]
    els = [("camera", 2, cam), ("vertex", n, vprops)]
    cases["mixed_int_skip"] = binary_file(els, [cam_rows, rows])
    # float coordinates (float32 x, double y, int z -> float cloud)
    fprops = [("x", "float"), ("y", "double"), ("z", "int"),
              ("red", "uchar"), ("green", "uchar"), ("blue", "uchar")]
    frows = [(float(np.float32(rng.normal())), float(rng.normal() * 100),
              int(rng.integers(-50, 50)), *[int(v) for v in rng.integers(0, 256, 3)])
             for _ in range(99)]
    cases["float_mixed"] = binary_file([("vertex", 99, fprops)], [frows])
    # uint32 coordinates at the top of the 21-bit range, char-typed coordinate
    uprops = [("red", "uchar"), ("green", "uchar"), ("blue", "uchar"),
              ("x", "uint"), ("y", "char"), ("z", "uint")]
    urows = [(*[int(v) for v in rng.integers(0, 256, 3)], int(rng.integers(0, 1 << 21)),
              int(rng.integers(0, 128)), (1 << 21) - 1) for _ in range(64)]
    cases["uint_top"] = binary_file([("vertex", 64, uprops)], [urows])
    # vertex element followed by a face list element (ignored)
    face = [("vertex_indices", "list uchar int")]
    hdr = header("binary_little_endian", [("vertex", 3, fprops[:0] + [
        ("x", "int"), ("y", "int"), ("z", "int"),
        ("red", "uchar"), ("green", "uchar"), ("blue", "uchar")]), ("face", 1, face)])
    body = b"".join(struct.pack("<iiiBBB", i, 2 * i, 3 * i, 10 * i, 20, 30) for i in range(3))
    cases["vertex_then_face"] = hdr + body + struct.pack("<Biii", 3, 0, 1, 2)
    # ascii with extra tokens, a comment and a skipped element
    ascii_hdr = header("ascii", [("camera", 1, cam), ("vertex", 4, [
        ("x", "int"), ("y", "int"), ("z", "int"), ("red", "uchar"),
        ("green", "uchar"), ("blue", "uchar"), ("quality", "float")])])
    cases["ascii_extra"] = ascii_hdr + b"1 2 3\n0 0 0 1 2 3 0.5\n5 6 7 255 0 9 1 extra\n" \
        b"1 1 1 0 0 0 0\n  2 3 4 5 6 7 8  \n"
    # CRLF line endings in the header
    cases["crlf_header"] = (b"ply\r\nformat binary_little_endian 1.0\r\nelement vertex 2\r\n"
                            b"property int x\r\nproperty int y\r\nproperty int z\r\n"
                            b"property uchar red\r\nproperty uchar green\r\n"
                            b"property uchar blue\r\nend_header\n"
                            + struct.pack("<iiiBBB", 1, 2, 3, 4, 5, 6)
                            + struct.pack("<iiiBBB", 7, 8, 9, 10, 11, 12))
    # a single point, all-zero coordinates (bit depth 1)
    cases["single_zero"] = binary_file([("vertex", 1, fprops[:0] + [
        ("x", "uint"), ("y", "uint"), ("z", "uint"), ("red", "uchar"), ("green", "uchar"),
        ("blue", "uchar")])], [[(0, 0, 0, 1, 2, 3)]])
    return cases


def error_cases():
    ok_props = [("x", "int"), ("y", "int"), ("z", "int"), ("red", "uchar"),
                ("green", "uchar"), ("blue", "uchar")]
    good = binary_file([("vertex", 2, ok_props)], [[(1, 2, 3, 4, 5, 6), (7, 8, 9, 1, 2, 3)]])
    cases = {
        "no_end_header": b"ply\nformat ascii 1.0\nelement vertex 0\n",
        "no_newline": b"ply\nformat ascii 1.0\nelement vertex 0\nend_header",
        "not_ply": b"plx\nformat ascii 1.0\nend_header\n",
        "bad_format_line": b"ply\nformat ascii\nend_header\n",
        "big_endian": b"ply\nformat binary_big_endian 1.0\nelement vertex 0\nend_header\n",
        "bad_element": b"ply\nformat ascii 1.0\nelement vertex\nend_header\n",
        "bad_count": b"ply\nformat ascii 1.0\nelement vertex 1.5\nend_header\n",
        "neg_count": b"ply\nformat ascii 1.0\nelement vertex -1\nend_header\n",
        "prop_first": b"ply\nformat ascii 1.0\nproperty int x\nend_header\n",
        "bad_list": b"ply\nformat ascii 1.0\nelement f 1\nproperty list uchar\nend_header\n",
        "bad_prop": b"ply\nformat ascii 1.0\nelement vertex 1\nproperty int\nend_header\n",
        "bad_type": b"ply\nformat ascii 1.0\nelement vertex 1\nproperty int64 x\nend_header\n",
        "unknown_kw": b"ply\nformat ascii 1.0\nfoo bar\nend_header\n",
        "no_format": b"ply\nelement vertex 0\nend_header\n",
        "no_vertex": b"ply\nformat ascii 1.0\nelement face 0\nend_header\n",
        "truncated": good[:-1],
        "missing_z": binary_file([("vertex", 1, ok_props[:2] + ok_props[3:])],
                                 [[(1, 2, 4, 5, 6)]]),
        "missing_blue": binary_file([("vertex", 1, ok_props[:5])], [[(1, 2, 3, 4, 5)]]),
        "wide_color": binary_file([("vertex", 1, ok_props[:3] + [
            ("red", "ushort"), ("green", "uchar"), ("blue", "uchar")])],
            [[(1, 2, 3, 4, 5, 6)]]),
        "negative": binary_file([("vertex", 2, ok_props)],
                                [[(1, 2, 3, 4, 5, 6), (7, -8, 9, 1, 2, 3)]]),
        "too_deep": binary_file([("vertex", 2, ok_props)],
                                [[(1, 2, 3, 4, 5, 6), (7, 1 << 22, 9, 1, 2, 3)]]),
        "vertex_list": b"ply\nformat binary_little_endian 1.0\nelement vertex 1\n"
                       b"property list uchar int idx\nend_header\n\x00",
        "skip_list": b"ply\nformat binary_little_endian 1.0\nelement f 1\n"
                     b"property list uchar int idx\nelement vertex 0\nproperty int x\n"
                     b"end_header\n\x00",
        "ascii_short_row": header("ascii", [("vertex", 1, ok_props)]) + b"1 2 3 4 5\n",
        "ascii_nan_token": header("ascii", [("vertex", 1, ok_props)]) + b"1 2 a 4 5 6\n",
        "ascii_range": header("ascii", [("vertex", 1, ok_props)]) + b"1 2 3 4 5 256\n",
        "ascii_truncated": header("ascii", [("vertex", 3, ok_props)]) + b"1 2 3 4 5 6\n",
        "ascii_negative": header("ascii", [("vertex", 1, ok_props)]) + b"1 -2 3 4 5 6\n",
        "empty_int": header("binary_little_endian", [("vertex", 0, ok_props)]),
        "empty_ascii_float": header("ascii", [("vertex", 0, [("x", "float"), ("y", "float"),
                                                             ("z", "float")] + ok_props[3:])]),
    }
    out = {}
    for name, data in cases.items():
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                fgbd.load_ply(data)
        except Exception as e:  # noqa: BLE001 -- recording the reference's behaviour
            out[name] = (data, type(e).__name__, str(e))
        else:
            raise SystemExit(f"error case {name} parsed without error")
    return out


def main():
    arrays, index = {}, {"save": {}, "load": {}, "errors": {}, "denoise": {}}

    def put(key, b):
        arrays[key] = np.frombuffer(b, np.uint8)

    clouds = {"quant21_edges": quant_edge_cloud(500, 21), "float_edges": float_cloud(300, 31)}
    for name, params, pc in synth_cases():
        clouds[name] = pc
        index["denoise"][name] = {"params": params}
    for name, pc in clouds.items():
        for fmt in ("binary", "ascii"):
            key = f"save/{name}/{fmt}"
            put(key, fgbd.save_ply(pc, fmt))
            index["save"][f"{name}/{fmt}"] = {"quantized": pc.is_quantized}
        arrays[f"cloud/{name}/coords"] = np.asarray(pc.coords)
        arrays[f"cloud/{name}/colors"] = np.asarray(pc.colors)
        index["save"][f"{name}/binary"]["bit_depth"] = pc.bit_depth
    for name, data in load_cases().items():
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            pc = fgbd.load_ply(data)
        put(f"load/{name}/file", data)
        arrays[f"load/{name}/coords"] = np.asarray(pc.coords)
        arrays[f"load/{name}/colors"] = np.asarray(pc.colors)
        index["load"][name] = {"bit_depth": pc.bit_depth,
                               "warnings": [str(x.message) for x in w]}
    for name, (data, cls, msg) in error_cases().items():
        put(f"errors/{name}", data)
        index["errors"][name] = {"exception": cls, "message": msg}
    cfg = fgbd.FilterConfig()
    for name in index["denoise"]:
        src = fgbd.save_ply(clouds[name], "binary")
        pc = fgbd.load_ply(src)
        out, rep = fgbd.denoise(pc, cfg)
        put(f"denoise/{name}/out", fgbd.save_ply(out, "binary"))
        arrays[f"denoise/{name}/colors"] = np.asarray(out.colors)
        index["denoise"][name].update(selected_q=rep.selected_q, sigma_est=rep.sigma_est)
        out2, _ = fgbd.denoise(pc, cfg, cached_q=3, cached_sigma_est=1.25)
        put(f"denoise/{name}/cached3", fgbd.save_ply(out2, "binary"))
        arrays[f"denoise/{name}/cached3_colors"] = np.asarray(out2.colors)
    np.savez_compressed(OUT / "ply.npz", **arrays)
    (OUT / "ply_index.json").write_text(json.dumps(index, indent=1, sort_keys=True))
    print(f"wrote {len(arrays)} arrays")


if __name__ == "__main__":
    main()
