"""Reference module name `polydet.pipeline` (pipeline.py): the entry points,
planning and forecast, re-exported from this package's executor/planner/predict."""

from .executor import resume, resume_report, run, run_report  # noqa: F401
from .planner import PipelineConfig, Plan, StageTimings, coefficient_bound, degree_bound, plan  # noqa: F401
from .predict import Prediction, predict, predicted_total  # noqa: F401
