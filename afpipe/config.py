"""afpipe.config — the reference's config API (pkg/src/afpipe/config.py:17-310), served by
this repo's mirror paper_2605_11005_b200.config: the same objects, not copies, so documents,
dataclasses and exceptions are interchangeable between the two names."""

from paper_2605_11005_b200.config import *  # noqa: F401,F403
from paper_2605_11005_b200.config import (  # noqa: F401
    ClusterConfig,
    ConfigError,
    Experiment,
    InvalidValue,
    MissingField,
    ModelConfig,
    ScheduleKind,
    SchemaViolation,
    Workload,
    load_experiment,
    parse_experiment,
    serialize_experiment,
    validate,
)
