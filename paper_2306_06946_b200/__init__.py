"""B200-native recursive corrective-motion contact solver (arXiv 2306.06946).

Drop-in for the hot path of the reference package ``contactnewton``
(/root/reference/pkg/src/contactnewton/__init__.py:13-60): the same public
names, backed by sm_100a kernels through the C ABI in include/cn_b200.h.
"""

from .errors import (
    ContactNewtonError,
    DegenerateFrameError,
    DegenerateTetError,
    DimensionMismatchError,
    InvalidAttachmentError,
    NonFiniteForceError,
    NotSPDError,
    ParseError,
    SingularBlockError,
    ValidationError,
)
from .mesh import TetMesh, box_mesh, five_tet_grid, load_mesh, save_mesh, surface_triangles
from .collision import (
    AttachKind,
    Attachment,
    ContactFrame,
    MeshGeometry,
    PairTable,
    PlaneGeometry,
    Pose,
    SphereGeometry,
    ProximityPair,
    build_frames,
    detect,
    max_frame_rotation,
    refresh_proximity,
    relinearize,
    signed_gaps,
)
from .constraints import (
    Delassus,
    DirectionMatrix,
    MappingDelassus,
    Violation,
    assemble_direction,
    assemble_H,
    assemble_W_standard,
    assemble_Wg,
    build_signed_mapping,
    compute_violation,
    fast_update_proximity,
    rebuild_W_fast,
)
from .linalg import Factorization, SparseSym, factorize, gemm, solve, solve_multi
from .solver import (
    LambdaState,
    NewtonConfig,
    PgsConfig,
    PgsResult,
    StepContext,
    local_solve,
    newton,
    newton_fast,
    newton_standard,
    pgs,
    regularize,
)

from .dynamics import (
    FreeMotion,
    MechanicalState,
    RigidBody,
    SoftBody,
    compute_free_motion,
    integrate_correction,
    lame_parameters,
    lumped_masses,
)
from .scene import (
    KinematicMeshSpec,
    MotionSpec,
    OutputConfig,
    PlaneSpec,
    RigidSphereSpec,
    SceneConfig,
    Simulation,
    Snapshot,
    SoftSpec,
    StepReport,
    load_scene,
    load_snapshot,
    run,
    save_snapshot,
    take_snapshot,
)

__version__ = "0.1.0"
