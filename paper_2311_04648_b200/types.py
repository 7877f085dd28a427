"""Data widths of the drop-in (mirrors grainforge/types.py:16-42).

Device layout (csrc/gf_common.cuh) on top of these: voxel u64 + sub-voxel
ushort4 (one 16-B record), quaternion float4, velocities VelT[4] (fp64 in the
parity build, fp32 in the throughput build), owner meta u32 = family << 24 |
mass-property template id, contact ids uint2 (kind in bits 30-31 of B), contact
history float4.
"""

import numpy as np

REAL = np.float32          # history, quaternions, geometry parameters
STATE_REAL = np.float64    # host-side owner kinematic state
SCRATCH = np.float64       # per-contact arithmetic
FAMILY = np.uint8
NUM_FAMILIES = 256
VOXEL_INDEX = np.uint64
SUBVOXEL = np.uint16
VOXEL_BITS_PER_AXIS = 21
SUBVOXEL_BITS = 16
VOXELS_PER_AXIS = 1 << VOXEL_BITS_PER_AXIS
SUBVOXELS_PER_EDGE = 1 << SUBVOXEL_BITS
INDEX = np.int64
MATERIAL_ID = np.uint8
BOUNDARY_MASS = 1.0e14
