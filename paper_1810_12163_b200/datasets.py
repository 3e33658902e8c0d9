"""Data formats either side of the hot path: the forest file and
7-Scenes-layout RGB-D sequences (SPEC.md bench_cli `load_dataset_sequence`).

* Forest file = the `serialize_forest` byte format that
  `scr_scene_create` parses; `save_forest` / `load_forest` / `Scene.from_file`-style helpers.
* A sequence directory holds `frame-NNNNNN.color.png` (8-bit RGB), `frame-NNNNNN.depth.png`
  (16-bit millimetres, 65535 = invalid) and `frame-NNNNNN.pose.txt` (4x4 row-major
  camera-to-world). Depth becomes metres; a pose that is non-rigid beyond 1e-3 is
  re-orthonormalised (with a warning), beyond 1e-1 it is rejected (MalformedPose); a
  missing pose leaves the frame without ground truth.

PNG is read and written with the standard library only (zlib), for the colour types the
layout uses: 8-bit RGB and 16-bit greyscale (non-interlaced, all five scanline filters).
"""
from __future__ import annotations

import glob
import os
import re
import struct
import warnings
import zlib
from dataclasses import dataclass, field

import numpy as np

from .native import MalformedData

INVALID_DEPTH_MM = 65535


class MissingFile(FileNotFoundError):
    pass


class MalformedPose(MalformedData):
    pass


# ---- forest file ---------------------------------------------------------------------------
def save_forest(path: str, blob: bytes) -> None:
    with open(path, "wb") as f:
        f.write(bytes(blob))


def load_forest(path: str) -> bytes:
    """Raw forest bytes; the format is validated by scr_scene_create (MalformedData)."""
    if not os.path.exists(path):
        raise MissingFile(path)
    with open(path, "rb") as f:
        return f.read()


# ---- PNG codec (stdlib) ----------------------------------------------------------------------
_SIG = b"\x89PNG\r\n\x1a\n"


def _chunk(tag: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + tag + data + struct.pack(">I", zlib.crc32(tag + data) & 0xFFFFFFFF)


def write_png(path: str, img: np.ndarray) -> None:
    """uint8 HxWx3 (RGB) or uint16 HxW (greyscale, big-endian in the file)."""
    if img.dtype == np.uint8 and img.ndim == 3 and img.shape[2] == 3:
        ctype, depth, raw = 2, 8, np.ascontiguousarray(img)
    elif img.dtype == np.uint16 and img.ndim == 2:
        ctype, depth, raw = 0, 16, np.ascontiguousarray(img.astype(">u2"))
    else:
        raise ValueError("write_png: uint8 HxWx3 or uint16 HxW")
    h, w = img.shape[:2]
    rows = raw.reshape(h, -1).view(np.uint8)
    data = b"".join(b"\x00" + rows[y].tobytes() for y in range(h))  # filter 0 per row
    ihdr = struct.pack(">IIBBBBB", w, h, depth, ctype, 0, 0, 0)
    with open(path, "wb") as f:
        f.write(_SIG + _chunk(b"IHDR", ihdr) + _chunk(b"IDAT", zlib.compress(data, 6)) + _chunk(b"IEND", b""))


def _paeth(a: int, b: int, c: int) -> int:
    p = a + b - c
    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
    return a if pa <= pb and pa <= pc else (b if pb <= pc else c)


def read_png(path: str) -> np.ndarray:
    if not os.path.exists(path):
        raise MissingFile(path)
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:8] != _SIG:
        raise MalformedData(f"{path}: not a PNG")
    off, idat, hdr = 8, [], None
    while off < len(buf):
        (n,) = struct.unpack(">I", buf[off:off + 4])
        tag, data = buf[off + 4:off + 8], buf[off + 8:off + 8 + n]
        off += 12 + n
        if tag == b"IHDR":
            hdr = struct.unpack(">IIBBBBB", data)
        elif tag == b"IDAT":
            idat.append(data)
        elif tag == b"IEND":
            break
    if hdr is None:
        raise MalformedData(f"{path}: no IHDR")
    w, h, depth, ctype, _, _, interlace = hdr
    if interlace:
        raise MalformedData(f"{path}: interlaced PNG not supported")
    chans = {0: 1, 2: 3, 4: 2, 6: 4}.get(ctype)
    if chans is None or depth not in (8, 16):
        raise MalformedData(f"{path}: colour type {ctype} / depth {depth} not supported")
    bpp = chans * depth // 8
    stride = w * bpp
    raw = zlib.decompress(b"".join(idat))
    out = np.zeros((h, stride), np.uint8)
    prev = np.zeros(stride, np.int32)
    pos = 0
    for y in range(h):
        ft = raw[pos]
        line = np.frombuffer(raw, np.uint8, stride, pos + 1).astype(np.int32)
        pos += 1 + stride
        if ft == 0:
            cur = line
        elif ft == 2:
            cur = (line + prev) & 255
        else:  # 1 (sub), 3 (average), 4 (paeth): left-dependent, byte by byte
            cur = np.zeros(stride, np.int32)
            for i in range(stride):
                a = cur[i - bpp] if i >= bpp else 0
                b = prev[i]
                c = prev[i - bpp] if i >= bpp else 0
                pred = a if ft == 1 else ((a + b) >> 1 if ft == 3 else _paeth(a, b, c))
                cur[i] = (line[i] + pred) & 255
        out[y] = cur
        prev = cur
    if depth == 16:
        img = out.view(">u2").astype(np.uint16).reshape(h, w, chans)
    else:
        img = out.reshape(h, w, chans)
    return img[:, :, 0] if chans == 1 else img[:, :, :3]


# ---- sequences --------------------------------------------------------------------------------
@dataclass
class SequenceSource:
    depths: list = field(default_factory=list)   # float32 metres (0 = invalid)
    rgbs: list = field(default_factory=list)     # uint8 HxWx3
    poses: list = field(default_factory=list)    # 4x4 camera->world or None (no ground truth)

    def __len__(self) -> int:
        return len(self.depths)


def _rigidify(M: np.ndarray, path: str) -> np.ndarray:
    R = M[:3, :3]
    dev = float(np.abs(R.T @ R - np.eye(3)).max())
    if dev > 1e-1 or abs(M[3] - [0, 0, 0, 1]).max() > 1e-1:
        raise MalformedPose(f"{path}: not a rigid transform (deviation {dev:.3g})")
    if dev > 1e-3:
        warnings.warn(f"{path}: pose re-orthonormalised (deviation {dev:.3g})")
        U, _, Vt = np.linalg.svd(R)
        R = U @ Vt
        if np.linalg.det(R) < 0:
            U[:, 2] *= -1
            R = U @ Vt
        M = M.copy()
        M[:3, :3] = R
        M[3] = [0, 0, 0, 1]
    return M


def load_dataset_sequence(directory: str) -> SequenceSource:
    if not os.path.isdir(directory):
        raise MissingFile(directory)
    ids = sorted({int(m.group(1)) for f in os.listdir(directory)
                  if (m := re.match(r"frame-(\d{6})\.depth\.png$", f))})
    seq = SequenceSource()
    for i in ids:
        stem = os.path.join(directory, f"frame-{i:06d}")
        d = read_png(stem + ".depth.png")
        if d.dtype != np.uint16:
            raise MalformedData(f"{stem}.depth.png: expected 16-bit depth")
        depth = np.where(d == INVALID_DEPTH_MM, 0.0, d.astype(np.float64) / 1000.0).astype(np.float32)
        rgb = read_png(stem + ".color.png")
        if rgb.ndim != 3 or rgb.dtype != np.uint8:
            raise MalformedData(f"{stem}.color.png: expected 8-bit RGB")
        pose = None
        if os.path.exists(stem + ".pose.txt"):
            M = np.loadtxt(stem + ".pose.txt", dtype=np.float64)
            if M.shape != (4, 4):
                raise MalformedPose(f"{stem}.pose.txt: expected a 4x4 matrix")
            pose = _rigidify(M, stem + ".pose.txt")
        seq.depths.append(depth)
        seq.rgbs.append(rgb)
        seq.poses.append(pose)
    return seq


def export_sequence(directory: str, depths, rgbs, poses=None) -> None:
    """Writes frames in the same layout (depth rounded to millimetres; 0 / invalid -> 65535)."""
    os.makedirs(directory, exist_ok=True)
    for i, (d, c) in enumerate(zip(depths, rgbs)):
        stem = os.path.join(directory, f"frame-{i:06d}")
        d = np.asarray(d, np.float64)
        valid = np.isfinite(d) & (d > 0) & (np.rint(d * 1000.0) < INVALID_DEPTH_MM)
        mm = np.where(valid, np.rint(np.where(valid, d, 0) * 1000.0), INVALID_DEPTH_MM).astype(np.uint16)
        write_png(stem + ".depth.png", mm)
        write_png(stem + ".color.png", np.asarray(c, np.uint8))
        if poses is not None and poses[i] is not None:
            np.savetxt(stem + ".pose.txt", np.asarray(poses[i], np.float64).reshape(4, 4), fmt="%.17g")


def pose_matrix(p) -> np.ndarray:
    """4x4 camera->world from an scr_pose / (R, t)."""
    from .relocaliser import pose_arrays, to_pose

    R, t = pose_arrays(to_pose(p))
    M = np.eye(4)
    M[:3, :3], M[:3, 3] = R, t
    return M
