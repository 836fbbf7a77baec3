"""GPU: the reference's metrics tests (pkg/tests/test_metrics.py:41-117,183-199)
restated against this package.  compute_metrics runs on the device metrics
kernels, and the round trip replays on the device.  The host-only ones
(nearest_rank, perturb_profiles) run unchanged against the mirror on CPU
(tests/test_reference_suite.py)."""
import pytest

from paper_2604_28175_b200 import PriorityLevel, compute_metrics

pytestmark = pytest.mark.gpu


def request_row(rid, priority="high", arrival=0.0, completion=5.0, deadline=10.0, dropped=0):
    violated = 1 if dropped or (completion != "" and completion > deadline) else 0
    return {"request": rid, "model": "m", "priority": priority, "arrival": arrival, "deadline_abs": deadline,
            "batch": "b0" if not dropped else "", "completion": "" if dropped else completion,
            "latency": "" if dropped else completion - arrival, "dropped": dropped, "violated": violated}


def test_all_meet():
    report = compute_metrics([request_row(f"r{i}") for i in range(10)])
    assert report.per_class[PriorityLevel.HIGH].violation_rate_pct == 0.0


def test_late_plus_dropped():
    rows = [request_row(f"ok{i}", completion=5.0) for i in range(95)]
    rows += [request_row(f"late{i}", completion=12.0) for i in range(3)]
    rows += [request_row(f"drop{i}", dropped=1) for i in range(2)]
    cm = compute_metrics(rows).per_class[PriorityLevel.HIGH]
    assert cm.arrivals == 100 and cm.violations == 5
    assert cm.violation_rate_pct == pytest.approx(5.0)


def test_dropped_excluded_from_latency():
    cm = compute_metrics([request_row("a", completion=4.0), request_row("b", dropped=1)]).per_class[PriorityLevel.HIGH]
    assert cm.p50_latency == 4.0 and cm.completed == 1


def test_goodput_windows():
    rows = [request_row("a", completion=500.0, deadline=1e6), request_row("b", completion=1500.0, deadline=1e6),
            request_row("c", completion=1600.0, deadline=1e6), request_row("late", completion=1700.0, deadline=1.0)]
    cm = compute_metrics(rows, window_ms=1000.0).per_class[PriorityLevel.HIGH]
    assert cm.goodput_counts == [1, 2]
    assert sum(cm.goodput_counts) + cm.violations == cm.arrivals


def test_partial_flag():
    rows = [request_row("a"), {"request": "pending", "model": "m", "priority": "high", "arrival": 0.0,
                               "deadline_abs": 10.0, "batch": "b1", "completion": "", "latency": "", "dropped": 0,
                               "violated": 0}]
    assert compute_metrics(rows).partial is True


def test_kernel_overhead_formula():
    batch = {"isolated_kernel": 4.0, "measured_kernel": 6.0, "est_latency": 10.0, "actual_latency": 8.0}
    report = compute_metrics([], batch_rows=[batch])
    assert report.kernel_overhead == [pytest.approx(0.5)]
    assert report.latency_error == [pytest.approx((10.0 - 8.0) / 8.0)]


def test_intf_error_signed():
    report = compute_metrics([], feedback_rows=[{"predicted": 1.2, "actual": 1.5}, {"predicted": 2.0, "actual": 1.6}])
    assert report.intf_error[0] == pytest.approx((1.2 - 1.5) / 1.5)
    assert report.intf_error[1] == pytest.approx(0.25)


def test_recomputed_metrics_identical(tmp_path):
    from paper_2604_28175_b200 import ExperimentConfig, WorkloadSpec, default_ground_truth, default_profiles, run
    from paper_2604_28175_b200.report import report_from_run_dir, write_run_dir
    from paper_2604_28175_b200.workload import ModelWorkload

    cfg = ExperimentConfig(profiles=default_profiles(),
                           workload=WorkloadSpec(duration_ms=800.0, models={"resnet50": ModelWorkload("poisson", 300.0),
                                                                            "vgg19": ModelWorkload("poisson", 200.0)}),
                           ground_truth=default_ground_truth(0.05), n_gpus=1, seed=5)
    result = run(cfg)
    write_run_dir(result, tmp_path / "run")
    recomputed = report_from_run_dir(tmp_path / "run", window_ms=result.metrics.window_ms)
    assert recomputed.to_dict() == result.metrics.to_dict()
