"""B200-native (sm_100a) implementation of MQ-GNN's per-iteration GraphSAGE
training path behind the reference ``mqpipe`` sampler/trainer API.

Compute runs in hand-written CUDA kernels reached through the C-ABI library
``libmqgnn.so`` (include/mqgnn.h); there is no CPU fallback.
"""

from .graph import DeviceGraph, build_csr, load
from .cache import (DeviceCache, RefreshStream, cache_probs_degree, cache_probs_walk,
                    gather_features, lookup, refresh_cache, refresh_mask,
                    weighted_sample_without_replacement)
from .samplers import (Block, MiniBatch, PhiloxStream, SamplerParams, SamplingError,
                       build_minibatch, node_wise_block, sample_node_wise)
from .layerwise import LayerBlock, fastgcn_probs, sample_fastgcn, sample_ladies
from .nn import (ModelState, accuracy, adam_step, backward, batch_loss, evaluate, forward,
                 full_forward, gcn_forward, init_model,
                 loss_and_grads, sage_forward, sgd_step)
from .racom import (DistExchange, LocalExchange, WindowDriver, apply_update, compute_sync_period,
                    staleness_cost, sync_models)
from .pipeline import STAGES, PipelineStopped, PipelineTimeout, Trace, TraceEvent, utilization
from .runtime import (EpochStats, PipelineConfig, batch_rng, plan_epoch, run_epoch,
                      transfer_stage)
from .trainer import PeerTimeout, StepRunner
from .peer import PeerExchange
from .autotune import (AutotuneError, auto_queue_depth, compute_cap, compute_queue_size,
                       steady_slice)

__version__ = "0.1.0"
