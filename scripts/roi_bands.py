"""Row-band overlap of the z-slab partition: per rank, the
stage-1 region of interest (the pixel rectangles its slab projects into, as the
library plans them) for C4 (512^3, 16 cameras at 1920x1080) at N = 1, 2, 4, 8,
and the per-rank NVLink egress of the bitmask exchange per frame (fused peer
stores: (N - 1) x the slab's words; NVLS multicast: 1 x).  Needs a GPU (the
library plans the ROI on a live handle)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_6811_b200 import from_scene  # noqa: E402
from synth.scene import make_scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
s = make_scene(name)
g = s.grid
full_px = int((s.widths.astype(np.int64) * s.heights).sum())
words_bytes = g.nwords * 4
out = {"config": name, "image_pixels_all_cameras": full_px, "bitmask_bytes_per_frame": words_bytes}
for N in (1, 2, 4, 8):
    ranks = []
    for r in range(N):
        rec = from_scene(s, rank=r, world=N)
        roi = rec.roi()
        px = int(((roi[:, 1] - roi[:, 0]).astype(np.int64) * (roi[:, 3] - roi[:, 2])).sum())
        ranks.append(px)
        rec.close()
    slab_bytes = words_bytes // N
    out[f"N{N}"] = {
        "roi_pixels_per_rank": ranks,
        "max_roi_fraction_of_images": max(ranks) / full_px,
        "sum_roi_over_single_gpu_roi": sum(ranks) / out["N1"]["roi_pixels_per_rank"][0] if N > 1 else 1.0,
        "egress_bytes_per_frame_fused_peer": (N - 1) * slab_bytes,
        "egress_bytes_per_frame_nvls": slab_bytes if N > 1 else 0,
        "egress_us_per_frame_fused_peer_at_770GBs": (N - 1) * slab_bytes / 770e9 * 1e6,
        "egress_us_per_frame_nvls_at_770GBs": (slab_bytes if N > 1 else 0) / 770e9 * 1e6,
    }
print(json.dumps(out, indent=1))
