"""B200-native AVEC destination-side execution path (arXiv 2103.04930).

The hot path lives in libavec_cuda.so (include/avec_cuda.h, sm_100a kernels)
and libavec_host.so / bin/avec-server (C++ wire server). This Python package is
the host-side mirror of the reference plugin interface over that C-ABI.
"""
from .backend import (B200Backend, Dims, Frame, Heatmap, ModelDescriptor, ModelHandle,  # noqa: F401
                      PinnedBuffer, PipelineStream, assemble_people, coco_limbs, device_count, make_model, model_digest,
                      output_elems, synth_posenet_weights)
from ._lib import AvecError, AvecLibraryMissing  # noqa: F401
