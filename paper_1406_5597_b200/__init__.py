"""paper_1406_5597_b200 — B200-native transpose-free slab 3D real FFT.

Drop-in for the STRIDED path of the reference ``slabfft`` package
(plan / forward / inverse with the STRIDED_INPLACE spectral layout); the
transforms run in hand-written sm_100a CUDA (libtffft.so) behind a C ABI.
"""

from .dfft import (DTYPES, FftPlan, forward, forward_many, gather_real, gather_spectral, inverse, inverse_many,
                   plan, scatter_real, scatter_spectral)
from .errors import (ConfigurationError, ConsistencyError, ContractError, CudaError, LayoutError,
                     ProtocolError, SizeError, SlabFftError, TransportError)
from .exchange import ExchangeOp, Strategy, exchange_schedule
from .streaming import HostPairStream
from .fields import forward_batch, inverse_batch, radial_wavenumber, turbulence_spectra, turbulence_spectrum
from .layout import (DistAxis, GlobalGrid, RealSlab, SlabLayout, SpectralSlab, SpectralTag,
                     TwoLevelStride, column_stride_descriptor, owned_range, spectral_offset, validate)
from .transport import (CommMode, CommPattern, CopyCounter, Endpoint, allgather_handles, init_ipc_endpoint,
                        init_nccl_endpoint, make_communicators, nccl_loopback, run_spmd)

__version__ = "0.1.0"
