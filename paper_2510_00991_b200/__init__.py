"""iccl-b200: B200-native implementation of ICCL's (arXiv 2510.00991) P2P hot path.

send/recv, batched isend/irecv and alltoall(v) move bytes zero-copy from the
caller's tensor into the peer GPU's tensor over NVLink 5 / NVSwitch: copy
engines (0 SMs) enqueued on the caller's stream behind stream memory
operations, hand-written sm_100a kernels for small / mid-size messages, the
backup path, and the MoE dispatch / combine fused with the alltoallv (K8 /
K10).  Primary-backup path failover resumes mid-message at the receiver's
breakpoint (driven by a watchdog thread that makes no CUDA call), and a
window monitor records every chunk's WR/WC pair.

The compute path lives in ``libiccl_b200.so`` (C ABI: ``include/iccl_b200.h``);
this package is its Python surface, mirroring the reference API
(``/root/reference/SPEC.md`` verbs / transport / monitor / collectives).
"""
from ._lib import LIB_PATH, lib  # noqa: F401  (fails loudly if the CUDA library is missing)
from .comm import Communicator, P2POp, Work, init  # noqa: F401
from .config import IcclConfig, retry_timeout  # noqa: F401
from .errors import (Aborted, ConfigError, ConnectionFailed, GroupTooSmall, IcclError, IcclTimeout,  # noqa: F401
                     InvalidArgument, InvalidConfig, NoSmAvailable, NonPositiveDuration, QpInErrorState,
                     SizeMismatch, TargetQpDead, UnknownWr, UnregisteredRegion, WindowNotFull, ZeroLengthMessage)
from .faults import FaultEntry, FaultScript  # noqa: F401
from .monitor import (MessageRecord, Monitor, ThroughputSample, detect_lagging_rank,  # noqa: F401
                      per_message_throughput, resample, sample_series, window_throughput)
from .moe import (DispatchPlan, config4_routing, config4_tokens, expand_rows, gather_rows, moe_combine,  # noqa: F401
                  moe_combine_fused, moe_dispatch, moe_dispatch_fused, plan_dispatch, scatter_rows)

__version__ = "0.1.0"
