"""Write tests/golden/full_material_digests.json: SHA-256 digests of the ORACLE's BC words of every block
row of the full-size 4k materials (C3, C4, C3'), in chunks of 64 block rows per texture.

Imports only oracle/ and synth/ (the seeded input generator): no value here comes from the CUDA path.
tests/test_gpu_parity.py::test_full_material_digests decodes the same materials on the GPU and compares
every chunk's digest, i.e. all 5.24 M (C3) / 8.39 M (C4) / 6.29 M (C3') words bit for bit, at the cost
of a one-time oracle run (about 10 minutes per material on 8 host cores).

usage: python tools/gen_golden_digests.py [config ...]   (default 3 4 6)
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

CHUNK_ROWS = 64
OUT = os.path.join(ROOT, "tests", "golden", "full_material_digests.json")


def digests(cfg: int) -> dict:
    W, H, spec = synth.config_shape(cfg)
    blob = synth.model_blob(cfg)
    om = oracle.Model(blob)
    BH = H // 4
    rec = {"config": cfg, "width": W, "height": H, "fmts": om.fmts, "chunk_rows": CHUNK_ROWS,
           "model_sha256": hashlib.sha256(blob).hexdigest(), "chunks": []}
    t0 = time.time()
    for r0 in range(0, BH, CHUNK_ROWS):
        r1 = min(BH, r0 + CHUNK_ROWS)
        words = om.decode_material(W, H, r0, r1)       # [tex][rows][BW] uint64, little-endian
        rec["chunks"].append([hashlib.sha256(words[k].astype("<u8").tobytes()).hexdigest() for k in range(om.n_tex)])
        print(f"C{cfg} rows [{r0},{r1}) {time.time() - t0:.0f}s", flush=True)
    rec["oracle_seconds"] = round(time.time() - t0, 1)
    return rec


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [3, 4, 6]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["_about"] = ("SHA-256 of the oracle's BC words (uint64 little-endian, [rows][BW]) per texture per "
                      f"{CHUNK_ROWS}-row chunk; written by tools/gen_golden_digests.py (oracle/ + synth/ only)")
    for cfg in cfgs:
        data[str(cfg)] = digests(cfg)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1)


if __name__ == "__main__":
    main()
