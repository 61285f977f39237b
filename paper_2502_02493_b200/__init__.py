"""B200-native EasySpec decode loop (arXiv 2502.02493).

The product is ``libespec_b200.so`` (C ABI: ``include/espec_c.h``), a C++ host
orchestrator over hand-written sm_100a kernels; ``espec`` is its Python
binding mirroring the reference's ``generate`` / stage API.
"""
from . import espec  # noqa: F401
from .espec import (BF16, F32, Engine, EspecError, ModelConfig, RunConfig, parse_plan_override,  # noqa: F401
                    plan_groups, tiny_config, tokenize, truncated_pair)
