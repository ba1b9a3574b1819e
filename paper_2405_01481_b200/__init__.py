"""B200-native PPO experience making (NeMo-Aligner, arXiv 2405.01481).

The product is ``libppoexp.so`` (sm_100a CUDA kernels + C++ host runtime behind
the C ABI in ``include/ppoexp.h``); ``ppoexp`` is the Python host mirror of
the reference's interfaces over that ABI.
"""
from . import ppoexp  # noqa: F401
from .ppoexp import (  # noqa: F401
    BF16, F32, ContractError, Context, DeviceModel, Engine, EngineOptions, ExperienceMaker, GenTask, GenerateResult,
    IndexError_, ModelConfig, PpoError, PpoHyper, RefitError, RolloutSeq, SamplingSpec, ShapeError, build_engine,
    expected_names, flat_to_params, reward_head, sequence_logprobs, shape_gae, value_estimates)
