"""Strait (arXiv 2604.28175) estimator + dispatch on NVIDIA B200 (sm_100a).

The public names mirror the reference package ``infersim`` (its
``__init__.py:44-91``) for the hot path: the interference predictor with its
online refit, the PCIe FIFO link, the priority-aware dispatch and the
trace-replay simulator.  All of their arithmetic runs in the in-tree CUDA
library ``_strait.so`` through the C-ABI declared in ``include/strait.h``;
there is no CPU fallback.
"""
from ._abi import SimulationOrderError, StraitUnavailable
from .domain import (Batch, ModelProfile, PriorityLevel, Request, ThroughputTimeline, time_weighted_average,
                     validate_profile)
from .pcie import PcieLinkState
from .predictor import (FeedbackSample, InterferencePredictor, OptimizerState, PredictorParams, UpdateResult,
                        estimate_latency, interference_degree, kernel_delay, kernel_effect, predict_interference,
                        pressure_exponent)
from .profiles import default_profiles, load_profile, random_profile, save_profile
from .runtime import AimdState, GpuRuntimeState, RunningTaskEntry
from .scheduler import (BatchPlan, PredictivePolicy, ScheduleDecision, SchedulingPolicy, TaskQueue, check_meet,
                        check_violate, complete_batch, early_drop, largest_feasible, make_policy, run_scheduling_pass,
                        submit_plan)
from .simulation import SimResult, Simulation, run, run_many
from .config import ExperimentConfig, GroundTruthParams, default_ground_truth, load_config
from .ground_truth import ground_truth_slowdown
from .metrics import MetricsReport, compute_metrics, perturb_profiles
from .workload import WorkloadSpec, gen_poisson, gen_uniform, load_trace

__version__ = "0.1.0"
