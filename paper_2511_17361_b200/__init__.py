"""B200-native superquadric voxelization (SuperQuadricOcc, arXiv 2511.17361).

Drop-in for the reference's voxelize / metrics path over
hand-written sm_100a kernels in libsqv.so (include/sqv.h).  See DESIGN.md.
"""
from .core import (EPS_MAX, EPS_MIN, F_CAP, ClassTable, PrimitiveBatch, Scene, SuperQuadric,
                   quat_to_matrix)
from .voxelize import (DenseGrids, SemanticGrid, VoxelGridSpec, VoxelizeConfig, VoxelizeResult,
                       Voxelizer, finalize, voxelize, voxelize_bruteforce)
from .metrics import miou, ray_iou, voxel_iou

__all__ = [
    "EPS_MIN", "EPS_MAX", "F_CAP", "SuperQuadric", "ClassTable", "Scene", "PrimitiveBatch",
    "quat_to_matrix", "VoxelGridSpec", "VoxelizeConfig", "DenseGrids", "SemanticGrid",
    "VoxelizeResult", "Voxelizer", "voxelize", "voxelize_bruteforce", "finalize",
    "voxel_iou", "miou", "ray_iou",
]
