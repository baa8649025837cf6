"""CPU pins for the checkpoint format helpers (tests/support/lshb_format.py)."""
from support.lshb_format import crc32c, crc32c_fast


def test_crc32c_standard_check_value():
    # CRC-32C check value (RFC 3720 / iSCSI; "123456789" -> 0xE3069283)
    assert crc32c(b"123456789") == 0xE3069283
    assert crc32c(b"") == 0
    assert crc32c(bytes(32)) == 0x8A9136AA          # RFC 3720 B.4: 32 bytes of zeros


def test_fast_crc_matches_bitwise():
    import os
    for n in (0, 1, 7, 100, 5000):
        d = os.urandom(n)
        assert crc32c_fast(d) == crc32c(d)
