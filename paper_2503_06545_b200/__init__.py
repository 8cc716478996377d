"""B200-native QuantCache accelerated DiT sampling path (arXiv 2503.06545).

Drop-in for the reference `ditrt` package's forward-and-sample path: the same
public names (DiTConfig, ThresholdConfig, Toggles, Scheduler, QuantRuntime,
generate, run_single, compute_minmax_params, quantize, matmul_int, ...), with
every hot-path computation in hand-written sm_100a kernels (libqcb200.so,
C ABI in include/qcb200.h).  There is no CPU fallback."""

from .errors import BudgetError, ConfigurationError, DimensionError, TraceFormatError
from .model import (QUANT_SITES, BlockCost, BlockWeights, DiTConfig, DiTModel, LayerHooks,
                    block_mac_cost, head_mac_cost, init_model, load_weights, save_weights,
                    timestep_embedding, weight_checksum)
from .schedule import (FP_BITS, ScheduleDecision, Scheduler, ThresholdConfig, Toggles,
                       TraceRecord, activation_bits, adapt_prune_rate, billed_macs,
                       prune_draw, prune_probability, redundancy_metric, refresh_interval)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent modules load lazily so `import paper_2503_06545_b200` stays
    # cheap for config / trace tooling.
    import importlib
    lazy = {
        "QuantCacheEngine": "engine", "EngineOptions": "engine",
        "QuantRuntime": "runtime",
        "NoiseSchedule": "sampler", "linear_beta_schedule": "sampler", "generate": "sampler",
        "reverse_step": "sampler", "final_step": "sampler", "forward_noise": "sampler",
        "QuantParams": "quant", "QuantizedTensor": "quant", "compute_minmax_params": "quant",
        "quantize": "quant", "dequantize": "quant", "balance_channels": "quant",
        "BalanceTransform": "quant", "allocate_weight_bits": "quant",
        "WeightBitPlan": "quant",
        "matmul_int": "tensor", "matmul_fp": "tensor", "mm": "tensor", "attention": "tensor",
        "layernorm": "tensor", "Tensor": "tensor", "divergence_score": "tensor",
        "layer_similarity": "tensor", "cumulative_variation": "tensor",
        "predict_noise": "forward", "block_forward": "forward",
        "RunConfig": "harness", "RunMetrics": "harness", "CalibrationData": "harness",
        "parse_config": "harness", "load_config": "harness", "run_single": "harness",
        "run_benchmark": "harness", "compare_outputs": "harness", "export_trace": "harness",
        "import_trace": "harness", "replay_check": "harness", "load_calibration": "harness",
        "save_calibration": "harness", "calibrate": "harness", "measure_sensitivity": "harness",
    }
    if name in lazy:
        mod = importlib.import_module(f".{lazy[name]}", __name__)
        return getattr(mod, name)
    raise AttributeError(name)
