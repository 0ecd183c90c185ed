"""B200-native PSFS voxel reconstruction (arXiv 1311.6811, section 2.2.2).

The hot path runs in the sm_100a kernels of ``libpsfs.so`` behind the C ABI
``include/psfs.h``; ``psfs`` is its thin ctypes binding and ``parallel`` the
multi-GPU plumbing (torch.distributed / NCCL).  Importing this package never
imports the CPU oracle.
"""
from .psfs import (MAX_BATCH, MAX_CAMERAS, PsfsError, Reconstructor, default_params,  # noqa: F401
                   from_scene, lib)
