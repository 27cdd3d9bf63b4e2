"""Run by tests/test_gpu_checked.py in a subprocess with NTBC_LIB=libntbc_checked.so (bounds checks +
shared-memory poisoning, NTBC_CHECKS=1): decodes a set of shapes / models and compares every word with the
oracle.  Argument: a tag printed back; the schedule (NTBC_NWG, NTBC_STATIC_SCHED) comes from the
environment, so the parent can require identical words under different schedules."""
import hashlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2407_09543_b200 import ntbc  # noqa: E402

assert ntbc.LIB_PATH.endswith("libntbc_checked.so"), ntbc.LIB_PATH


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def main():
    h = hashlib.sha256()
    cases = []
    W, H, _ = synth.config_shape(1)
    cases.append((synth.model_blob(1), W, H, (0, H // 4)))
    W, H, _ = synth.config_shape(2)
    cases.append((synth.model_blob(2), W, H, (126, 130)))
    for (w, hh) in ((4, 4), (12, 8), (4 * 129, 8), (4 * 300, 12), (4 * 256 + 4, 4)):
        sp = synth.ModelSpec([synth.BC1, synth.BC4, synth.BC4], hidden=32, block_levels=3, block_coarsest=8,
                             texel_levels=4, texel_coarsest=8)
        cases.append((synth.serialize(synth.random_model(sp, w * 7 + hh)), w, hh, (0, hh // 4)))
    sp = synth.ModelSpec([synth.BC1, synth.BC4], hidden=32, block_levels=3, block_coarsest=3, texel_levels=4,
                         texel_coarsest=5)
    cases.append((synth.serialize(synth.random_model(sp, 35)), 4 * 130, 36, (0, 9)))
    for fm, hid, nv in (([synth.BC4] * 8, 32, False), ([synth.BC1] * 8, 64, False), ([synth.BC1, synth.BC4] * 4, 64, True)):
        blob = synth.serialize(synth.random_model(synth.ModelSpec(list(fm), hidden=hid, naive=nv), len(fm) * 100 + hid))
        cases.append((blob, 4 * 300, 4 * 6, (0, 6)))
    for blob, w, hh, (r0, r1) in cases:
        m = ntbc.Model(blob)
        outs = ntbc.decode_material([m], w, hh)
        ref = oracle.Model(blob).decode_material(w, hh, r0, r1)
        for k in range(m.n_tex):
            g = u64(outs[k])
            assert np.array_equal(g[r0:r1], ref[k]), (w, hh, k)
            h.update(g.tobytes())
        # a row shard into 8-B aligned planes (8-byte stores)
        part = torch.zeros((m.n_tex, (r1 - r0) * (w // 4) + 2), dtype=torch.int64, device="cuda")
        ntbc.decode_material([m], w, hh, row_begin=r0, row_end=r1,
                             out_ptrs=[part[k].data_ptr() + 8 for k in range(m.n_tex)])
        for k in range(m.n_tex):
            got = u64(part[k])[1:1 + (r1 - r0) * (w // 4)].reshape(r1 - r0, w // 4)
            assert np.array_equal(got, ref[k]), ("shard", w, hh, k)
    # seeded random models and shapes (tests/fuzz_cases.py), shards into 8-B-only aligned planes included
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from fuzz_cases import cases as fuzz_cases
    for blob, w, hh, r0, r1, misalign in fuzz_cases(24, seed=77):
        m = ntbc.Model(blob)
        rows, bw = r1 - r0, w // 4
        buf = torch.full((m.n_tex, rows * bw + 2), -1, dtype=torch.int64, device="cuda")
        ntbc.decode_material([m], w, hh, row_begin=r0, row_end=r1,
                             out_ptrs=[buf[k].data_ptr() + (8 if misalign else 0) for k in range(m.n_tex)])
        ref = oracle.Model(blob).decode_material(w, hh, r0, r1)
        off = 1 if misalign else 0
        for k in range(m.n_tex):
            got = u64(buf[k])[off:off + rows * bw].reshape(rows, bw)
            assert np.array_equal(got, ref[k]), ("fuzz", w, hh, k)
            h.update(got.tobytes())
    # contract F (binary32 activations, hi/lo split operands) on seeded random non-naive models, vs the oracle's F mode
    n_f = 0
    for blob, w, hh, r0, r1, misalign in fuzz_cases(40, seed=91):
        om = oracle.Model(blob)
        if om.naive or n_f >= 8:
            continue
        n_f += 1
        m = ntbc.Model(blob)
        ntbc.set_contract(m, 1)
        outs = ntbc.decode_material([m], w, hh, row_begin=r0, row_end=r1)
        with oracle.contract_f():
            ref = om.decode_material(w, hh, r0, r1)
        for k in range(m.n_tex):
            assert np.array_equal(u64(outs[k]), ref[k]), ("contract F", w, hh, k)
            h.update(u64(outs[k]).tobytes())
    # contract P (binary16 selu arithmetic) on seeded random non-naive models, vs the oracle's P mode
    n_p = 0
    for blob, w, hh, r0, r1, misalign in fuzz_cases(40, seed=93):
        om = oracle.Model(blob)
        if om.naive or n_p >= 6:
            continue
        n_p += 1
        m = ntbc.Model(blob)
        ntbc.set_contract(m, 2)
        outs = ntbc.decode_material([m], w, hh, row_begin=r0, row_end=r1)
        with oracle.contract_p():
            ref = om.decode_material(w, hh, r0, r1)
        for k in range(m.n_tex):
            assert np.array_equal(u64(outs[k]), ref[k]), ("contract P", w, hh, k)
            h.update(u64(outs[k]).tobytes())
    # conservative pair (one launch, CTAs partitioned by model)
    rgb = synth.serialize(synth.random_model(synth.ModelSpec([synth.BC1, synth.BC1], block_levels=4, texel_levels=5), 5))
    sc = synth.serialize(synth.random_model(synth.ModelSpec([synth.BC4] * 4, block_levels=4, texel_levels=5), 6))
    outs = ntbc.decode_material([ntbc.Model(rgb), ntbc.Model(sc)], 256, 64)
    ref = list(oracle.Model(rgb).decode_material(256, 64)) + list(oracle.Model(sc).decode_material(256, 64))
    for k in range(6):
        assert np.array_equal(u64(outs[k]), ref[k]), ("pair", k)
        h.update(u64(outs[k]).tobytes())
    mr, ms = ntbc.Model(rgb), ntbc.Model(sc)          # the same pair under contract F (one launch)
    ntbc.set_contract(mr, 1)
    ntbc.set_contract(ms, 1)
    outs = ntbc.decode_material([mr, ms], 256, 64)
    with oracle.contract_f():
        ref = list(oracle.Model(rgb).decode_material(256, 64)) + list(oracle.Model(sc).decode_material(256, 64))
    for k in range(6):
        assert np.array_equal(u64(outs[k]), ref[k]), ("pair F", k)
    # the standalone pack kernel
    for fmts, BW, BH in (([1, 1, 4, 4, 4], 41, 13), ([4], 1, 1), ([1] * 4 + [4] * 4, 130, 3)):
        ep, col = synth.pack_inputs(fmts, BW, BH, seed=BW * 31 + BH)
        g = ntbc.pack(fmts, torch.from_numpy(ep).cuda(), torch.from_numpy(col).cuda(), 4 * BW, 4 * BH)
        o = oracle.pack(fmts, ep, col, 4 * BW, 4 * BH)
        for k in range(len(fmts)):
            assert np.array_equal(u64(g[k]), o[k]), ("pack", fmts, k)
    torch.cuda.synchronize()
    print("OK", sys.argv[1] if len(sys.argv) > 1 else "", h.hexdigest(), flush=True)


if __name__ == "__main__":
    main()
