"""Gather-probe sweep: 1, 2, 4 sectors per line x blocks per SM x table size (profiles/)."""
import ctypes as C, sys
sys.path.insert(0,'.')
from paper_1311_6811_b200 import psfs
L = psfs.lib()
for G in (1,2,4):
    for bps in (2,3,4,8):
        for mb in (32, 64):
            d = C.c_double()
            rc = L.psfs_probe_gather_bandwidth(mb<<20, G, bps, C.byref(d))
            print(G, bps, mb, rc, round(d.value/1e12,2), "TB/s", round(d.value/1965e6/148/32,3), "sectors/clk/SM")
