"""ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product path).

Pure-Python restatement of the reference's DOGS scene container and GSPL
checkpoint codec, used to check the native encoder / decoder byte for byte:

  container   scene_io.cpp:124-132 (encode_scene), :134-176 (decode_scene):
              b"DOGS", u32 version 1, then tagged sections (4-byte tag, u64
              payload length, payload), CAMS and PNTS always written, GSPL
              only with a checkpoint; unknown / repeated tags, trailing bytes
              inside a section and short payloads are FormatErrors.
  CAMS        scene_io.cpp:23-36 / 68-85: u64 count; per view u64 id, f64 fx fy
              cx cy, u32 width height, f64 quaternion[4], f64 translation[3],
              u32 path length + bytes (77 fixed bytes per view).
  PNTS        scene_io.cpp:38-46 / 87-95: u64 count; per point f32 xyz, u8 rgb.
  GSPL        scene_io.cpp:48-59 / 97-122: u64 count, u32 feature width (3 or
              12), u64 ids, f32 positions [n][3], rotations [n][4], log-scales
              [n][3], features [n][F], opacity logits [n]; ids strictly ascending.
  model.dogs  main.cpp:353-357: a container holding only the narrowed model.

Little-endian throughout (serial.hpp). Error codes: errors.hpp:10-19.
Parity anchor: the reference's own tests of this format (test_image_scene.cpp:
127-250, acceptance_main.cpp:640-680): byte-exact re-encode, exact f32
narrowing, and the error code of each malformed input.
"""
import struct

import numpy as np

CODES = ("BadMagic", "UnsupportedVersion", "TruncatedSection", "UnknownSection", "TruncatedBuffer",
         "CountOverflow", "NonMonotoneIds", "BadHeader")


class OracleFormatError(Exception):
    def __init__(self, code, msg=""):
        super().__init__(f"{code}: {msg}")
        self.code = code


def narrow(cloud):
    """narrow_to_f32 (scene_io.cpp:230-241): every parameter through float32."""
    out = dict(cloud)
    for k in ("pos", "rot", "ls", "feat", "op"):
        out[k] = np.asarray(cloud[k], np.float64).astype(np.float32).astype(np.float64)
    return out


def gspl_payload(cloud):
    ids = np.asarray(cloud["ids"], np.uint64)
    n = len(ids)
    fd = int(np.asarray(cloud["feat"]).reshape(n, -1).shape[1]) if n else int(cloud.get("fd", 3))
    parts = [struct.pack("<QI", n, fd), ids.astype("<u8").tobytes()]
    for k, w in (("pos", 3), ("rot", 4), ("ls", 3), ("feat", fd), ("op", 1)):
        parts.append(np.asarray(cloud[k], np.float64).reshape(n * w).astype("<f4").tobytes())
    return b"".join(parts)


def cams_payload(views):
    out = [struct.pack("<Q", len(views))]
    for v in views:
        path = v.get("path", "").encode()
        out.append(struct.pack("<Q4d2I4d3dI", v["id"], v["fx"], v["fy"], v["cx"], v["cy"], v["width"], v["height"],
                               *v["q"], *v["t"], len(path)))
        out.append(path)
    return b"".join(out)


def pnts_payload(points):
    out = [struct.pack("<Q", len(points))]
    for p in points:
        out.append(struct.pack("<3f3B", *p["pos"], *p["rgb"]))
    return b"".join(out)


def section(tag, payload):
    return tag + struct.pack("<Q", len(payload)) + payload


def encode_scene(views=(), points=(), checkpoint=None):
    b = b"DOGS" + struct.pack("<I", 1) + section(b"CAMS", cams_payload(views)) + section(b"PNTS", pnts_payload(points))
    if checkpoint is not None:
        b += section(b"GSPL", gspl_payload(checkpoint))
    return b


def encode_model(cloud):
    return encode_scene(checkpoint=narrow(cloud))


class _Reader:
    def __init__(self, data, code):
        self.d, self.at, self.code = data, 0, code

    def take(self, k):
        if k > len(self.d) - self.at:
            raise OracleFormatError(self.code, "read past end")
        b = self.d[self.at:self.at + k]
        self.at += k
        return b

    def unpack(self, fmt):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))

    def left(self):
        return len(self.d) - self.at


def _count(r, count, item):
    if count > r.left() // item:
        raise OracleFormatError("CountOverflow")
    return count


def decode_checkpoint(data):
    """decode_scene restricted to what the tests compare: the GSPL cloud (or
    None), after validating every section the way the reference does."""
    top = _Reader(data, "TruncatedBuffer")
    if top.take(4) != b"DOGS":
        raise OracleFormatError("BadMagic")
    (version,) = top.unpack("<I")
    if version != 1:
        raise OracleFormatError("UnsupportedVersion")
    seen, ckpt = set(), None
    while top.at != len(data):
        tag = top.take(4)
        (ln,) = top.unpack("<Q")
        if ln > top.left():
            raise OracleFormatError("TruncatedSection")
        sec = _Reader(top.take(ln), "TruncatedSection")
        if tag not in (b"CAMS", b"PNTS", b"GSPL"):
            raise OracleFormatError("UnknownSection")
        if tag in seen:
            raise OracleFormatError("BadHeader")
        seen.add(tag)
        if tag == b"CAMS":
            n = _count(sec, sec.unpack("<Q")[0], 77)
            for _ in range(n):
                *_, plen = sec.unpack("<Q4d2I4d3dI")
                sec.take(plen)
        elif tag == b"PNTS":
            n = _count(sec, sec.unpack("<Q")[0], 15)
            sec.take(15 * n)
        else:
            count, fd = sec.unpack("<QI")
            if fd not in (3, 12):
                raise OracleFormatError("BadHeader")
            n = _count(sec, count, 8 + 4 * (11 + fd))
            ids = np.frombuffer(sec.take(8 * n), "<u8").astype(np.uint64)
            arr = {}
            for k, w in (("pos", 3), ("rot", 4), ("ls", 3), ("feat", fd), ("op", 1)):
                a = np.frombuffer(sec.take(4 * w * n), "<f4").astype(np.float64)
                arr[k] = a.reshape(n, w) if w > 1 else a
            if n > 1 and np.any(ids[1:] <= ids[:-1]):
                raise OracleFormatError("NonMonotoneIds")
            ckpt = dict(ids=ids, **arr)
        if sec.at != len(sec.d):
            raise OracleFormatError("TruncatedSection")
    return ckpt
