"""Shared fixtures: the reference's small traces, golden loaders, GPU marker.

Mirrors the reference fixtures (reference tests/conftest.py:20-53): the
four-batch worked example {3,9},{3,4},{3,6},{1,6} numbered 1..4, and the
small Zipf(1.05) trace (2 tables 600/400, D=4, 60 batches of 64, seed 7).
Golden data under tests/golden/ was produced by the reference itself
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2202_12429_b200.traces import (  # noqa: E402
    Batch,
    EmbeddingKey,
    Example,
    Schema,
    ZipfSpec,
    batchify_columns,
    generate_columns,
)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def make_batch(iteration: int, row_ids: list, table_id: int = 0) -> Batch:
    """One single-table batch with one example per key (labels i & 1)."""
    return Batch(iteration, [Example(i & 1, (), (EmbeddingKey(table_id, r),)) for i, r in enumerate(row_ids)])


def unpack(packed: int) -> EmbeddingKey:
    return EmbeddingKey(packed >> 44, packed & ((1 << 44) - 1))


@pytest.fixture
def worked_trace() -> list:
    return [make_batch(1, [3, 9]), make_batch(2, [3, 4]), make_batch(3, [3, 6]), make_batch(4, [1, 6])]


@pytest.fixture(scope="session")
def small_schema() -> Schema:
    return Schema(2, (600, 400), 2, 4)


@pytest.fixture(scope="session")
def small_batches(small_schema) -> list:
    rows, labels, dense = generate_columns(ZipfSpec(small_schema, 1.05, 60 * 64, seed=7))
    return batchify_columns(rows, labels, dense, 64)


@pytest.fixture(scope="session")
def small_object_batches(small_batches) -> list:
    """Same trace, object-backed (exercises the Example-list path)."""
    return [Batch(b.iteration, list(b.examples)) for b in small_batches]
