"""Independent reader of SPEC's LSHB / LBF1 containers, used to
check lshbloom_save's output byte by byte.  CRC32C (Castagnoli, reflected polynomial
0x82F63B78) is computed bitwise here, independently of the library."""
import struct


def crc32c(data: bytes, crc: int = 0) -> int:
    crc ^= 0xFFFFFFFF
    for byte in data:
        crc ^= byte
        for _ in range(8):
            crc = (crc >> 1) ^ (0x82F63B78 & -(crc & 1))
    return crc ^ 0xFFFFFFFF


def _table():
    t = []
    for i in range(256):
        c = i
        for _ in range(8):
            c = (c >> 1) ^ (0x82F63B78 & -(c & 1))
        t.append(c)
    return t


_T = _table()


def crc32c_fast(data: bytes) -> int:
    """Table-driven CRC32C for large payloads (checked against crc32c() in tests)."""
    import numpy as np
    crc = 0xFFFFFFFF
    for byte in data if len(data) < 4096 else np.frombuffer(data, np.uint8).tolist():
        crc = _T[(crc ^ byte) & 0xFF] ^ (crc >> 8)
    return crc ^ 0xFFFFFFFF


def read_lshb(blob: bytes):
    """Parse and verify a container; returns (header dict, [filter dicts with 'payload'])."""
    o = 0
    hdr = {}
    magic, version, threshold, num_perm, b, r, sseed, bseed, n_docs, p_eff, doc_count = struct.unpack_from(
        "<4sIdIIIQQQdQ", blob, o)
    o += struct.calcsize("<4sIdIIIQQQdQ")
    hdr.update(magic=magic, version=version, threshold=threshold, num_perm=num_perm, b=b, r=r,
               signature_seed=sseed, band_hash_seed=bseed, n_docs=n_docs, p_effective=p_eff,
               doc_count=doc_count)
    filters = []
    for _ in range(b):
        start = o
        fm, fv, seed, cap, tp, m, k, inserted = struct.unpack_from("<4sIQQdQIQ", blob, o)
        o += struct.calcsize("<4sIQQdQIQ")
        n = (m + 7) // 8
        payload = blob[o:o + n]
        o += n
        (crc,) = struct.unpack_from("<I", blob, o)
        filters.append(dict(magic=fm, version=fv, seed=seed, capacity_n=cap, target_p=tp, m=m, k=k,
                            inserted=inserted, payload=payload, crc=crc, crc_ok=crc32c_fast(blob[start:o]) == crc))
        o += 4
    (crc,) = struct.unpack_from("<I", blob, o)
    hdr["crc_ok"] = crc32c_fast(blob[:o]) == crc
    hdr["size"] = o + 4
    return hdr, filters
