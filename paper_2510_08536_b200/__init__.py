"""B200-native drop-in for the reference package ``ldurepart`` — hot path only.

Repartitioned CPU-assembly -> GPU-solve (arXiv 2510.08536): ``repartition``
(create once), ``update`` (values only, every timestep) and ``cg_solve`` /
``spmv`` (distributed Krylov solve), with the reference's types, errors and
collective context.  Compute runs in libldurepart_b200.so (hand-written
sm_100a CUDA + C++ behind a C ABI, include/ldurepart_b200.h); PyTorch only
owns device and pinned host memory.  No CPU fallback exists.
"""

from .core import (MM_HEADER, CooMatrix, DeviceCooMatrix, DistributedCooMatrix, InterfaceBlock,
                   LduMatrix, PartitionMap, coo_from_entries, gpu_owner, ldu_to_coo,
                   make_partition_map, read_matrix_market, validate_ldu, write_matrix_market)
from .cavity import (StructuredGrid, SubdomainMesh, assemble_poisson, build_grid,
                     decompose_slab, perturb_coefficients, perturb_diag_into)
from .transport import (CAT_DEVICE_DIRECT, CAT_DEVICE_STAGED, CAT_RANK, CommGroup,
                        DeadlockError, DeviceBuffer, RankContext, RankFailedError, World,
                        WorldError, run_world, split_active)
from .solver import (HaloPlan, SolveReport, bicgstab_solve, build_halo_plan, cg_solve,
                     krylov_solve, pcg_solve, spmv)
from .repart import (RepartitionedSystem, ScatterMap, SparsityPattern, UpdatePattern,
                     build_scatter_map, build_update_pattern, dump_scatter, dump_sparsity,
                     exchange_patterns,
                     extract_sparsity, fuse_patterns, pack_order_pairs, repartition,
                     sparsity_fingerprint)
from .update import (PackedCoefficients, PatternDriftError, TRANSFER_MODES, apply_scatter,
                     capture_device_base, pack_coefficients, transfer_coefficients, update,
                     update_on_device)

__version__ = "0.1.0"
from .verify import gather_global, read_curves_csv, write_curves_csv  # noqa: E402
