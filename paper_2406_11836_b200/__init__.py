"""B200-native drop-in for the RetinaGS distributed 3DGS training step.

The product is libdgs_b200.so (sm_100a kernels + C-ABI, include/dgs_capi.h);
this package is the host-side mirror of the reference interface over it.
"""
from .capi import LIB_PATH, Camera, lib  # noqa: F401
from .engine import (Context, Manager, PartitionTable, Splats, assign_subsets, build_kdtree,  # noqa: F401
                     perturb, position_lr, render_options, ring_camera, synth_splats, train_config)
