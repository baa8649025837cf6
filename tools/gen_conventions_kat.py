"""Write tests/golden/conventions_kat.json: known-answer vectors of the documented conventions
(R1 fingerprint, R5 family, R3/R6 signature and band hash, R10 probes, and
the blocked variant's offsets).  Calls only oracle/ (never the CUDA path); the values are then
checked against the independent micro-oracle by tests/test_oracle_micro.py.

Usage: python tools/gen_conventions_kat.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def hx(v):
    return "%016x" % int(v)


def main():
    out = {"_source": "tools/gen_conventions_kat.py (oracle/ only); conventions: DESIGN.md section 3 "
                      "R1, R3-R6, R10 and section 5 (blocked offsets); pinned against "
                      "tests/support/micro_oracle.py",
           "fingerprint": [], "family": [], "signature": [], "probes": []}
    for ids in ([0], [0, 0], [1, 2, 3, 4, 5], [4294967295] * 5, [17, 5, 99], [0, 1, 2, 3, 4, 5, 6]):
        out["fingerprint"].append({"ids": ids, "fp": hx(oracle.fingerprint(ids))})
    for seed in (0, 42):
        a, b, c, d, s1, s2 = oracle.family(seed, 8, 8, 4)
        out["family"].append({"seed": seed, "a": [hx(x) for x in a], "b": [hx(x) for x in b],
                              "c": [hx(x) for x in c], "d": [hx(x) for x in d],
                              "s1": [hx(x) for x in s1], "s2": [hx(x) for x in s2]})
    doc = [3, 1, 4, 1, 5, 9, 2, 6, 5, 3, 5, 8, 9, 7, 9, 3, 2, 3, 8, 4]
    for seed, num_perm, b, r in ((0, 128, 16, 8), (0, 128, 20, 6), (7, 32, 4, 8)):
        sig = oracle.signature_doc(doc, num_perm, seed)
        bh = [oracle.band_hash(sig, j, r, seed) for j in range(b)]
        out["signature"].append({"ids": doc, "seed": seed, "num_perm": num_perm, "b": b, "r": r,
                                 "sig": sig.tolist(), "band_hashes": [hx(x) for x in bh]})
    _, _, _, _, s1, s2 = oracle.family(0, 0, 0, 2)
    bh = 0x0123456789ABCDE
    for m in (23_962_646, 23_962_645_944):
        g = oracle.probes(bh, int(s1[1]), int(s2[1]), m, 17)
        out["probes"].append({"blocked": False, "bh": hx(bh), "s1": hx(s1[1]), "s2": hx(s2[1]), "m": m,
                              "k": 17, "g": [int(x) for x in g]})
    for nb in (23_402, 23_401_022):
        g = oracle.probes_blocked(bh, int(s1[0]), int(s2[0]), nb, 17)
        out["probes"].append({"blocked": True, "bh": hx(bh), "s1": hx(s1[0]), "s2": hx(s2[0]), "nb": nb,
                              "k": 17, "g": [int(x) for x in g]})
    path = os.path.join(ROOT, "tests", "golden", "conventions_kat.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path)


if __name__ == "__main__":
    main()
