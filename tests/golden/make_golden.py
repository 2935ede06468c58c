"""Regenerate tests/golden/seq_small.npz from the UNMODIFIED reference build
(oracle/_ref/libcbi_ref.so). Run in the build container (needs /root/reference
to have built oracle/_ref):  python tests/golden/make_golden.py

Content: the scene-labeling layer list at 48x64 (derived dims), weights
fill_random_weights(seed 1), tau 0.05, a 6-frame gen_synthetic sequence, and
the reference's final retained output plus layer-1 index list per frame.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1808_05488_b200 import cbi  # noqa: E402
from tests import oracle  # noqa: E402


def main():
    seed, H, W, taus = 1, 48, 64, [0.05] * 5
    spec = cbi.make_seg_spec(seed, H, W)
    frames = oracle.ref_gen_synthetic(cbi.SyntheticConfig(H, W, 3, 6, 2, 10, 3, 3, 0.0, 77))
    net = oracle.RefNet(spec, taus)
    outs, idxs, counts = [], [], []
    l1 = net.shapes[0]
    for f in frames:
        outs.append(net.forward(f))
        m = net.stats(0)["map"]
        idx = np.argwhere(m).astype(np.int32)
        counts.append(len(idx))
        pad = np.zeros((l1[2] * l1[3], 2), np.int32)
        pad[:len(idx)] = idx
        idxs.append(pad)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "seq_small.npz"),
                        seed=seed, height=H, width=W, taus=np.array(taus, np.float32), frames=frames,
                        outputs=np.stack(outs), l1_idx=np.stack(idxs), l1_count=np.array(counts, np.int64))
    print("wrote seq_small.npz", np.stack(outs).shape, counts)


if __name__ == "__main__":
    main()
