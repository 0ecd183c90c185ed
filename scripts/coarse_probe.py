"""Coarse-pass probe (C2): per-kernel device times and fix-up counts for the
coarse and exact paths; used under ncu for the kernel captures in profiles/."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1311_6811_b200 import from_scene  # noqa: E402
from synth.scene import make_frames, make_scene  # noqa: E402


def main():
    nf = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    s = make_scene("C2")
    frames = torch.from_numpy(np.stack([make_frames(s, f % 16) for f in range(nf)])).cuda()
    for mode in (1, 0):
        rec = from_scene(s)
        rec.set_coarse(mode)
        rec.set_overlap(False, 0)
        _, B = rec.alloc_outputs(nf, logodds=False)
        rec.reconstruct_batch(frames, nf, bits=B)
        torch.cuda.synchronize()
        rec.coarse_status(reset=True)
        rec.set_profiling(True)
        for _ in range(reps):
            rec.reconstruct_batch(frames, nf, bits=B)
        torch.cuda.synchronize()
        t = rec.kernel_times(reset=True)
        _, nfix = rec.coarse_status(reset=True)
        print(f"mode {mode}: {t}  fixups/call {nfix / reps:.0f}", flush=True)


if __name__ == "__main__":
    main()
