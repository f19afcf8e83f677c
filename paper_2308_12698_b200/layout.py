"""Initial layouts for benches and tests (config.py:147-179 ``layout_poses``)."""

from __future__ import annotations

import numpy as np

from .errors import ValidationError


def layout_poses(layout: dict, count: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Initial positions and headings for ``count`` agents: grid / circle / random_box."""
    kind = layout.get("kind", "grid")
    if kind == "grid":
        spacing = float(layout.get("spacing", 2.0))
        origin = np.asarray(layout.get("origin", (0.0, 0.0, 5.0)), dtype=float)
        cols = max(1, int(np.ceil(np.sqrt(max(count, 1)))))
        idx = np.arange(count)
        pos = np.stack([(idx % cols) * spacing, (idx // cols) * spacing, np.zeros(count)], axis=1)
        pos += origin
        yaw = np.zeros(count)
    elif kind == "circle":
        radius = float(layout.get("radius", 5.0))
        z = float(layout.get("z", 5.0))
        center = np.asarray(layout.get("center", (0.0, 0.0)), dtype=float)
        phases = 2.0 * np.pi * np.arange(count) / max(count, 1)
        pos = np.stack([center[0] + radius * np.cos(phases), center[1] + radius * np.sin(phases),
                        np.full(count, z)], axis=1)
        yaw = phases + np.pi / 2
    elif kind == "random_box":
        low = np.asarray(layout.get("low", (0.0, 0.0, 2.0)), dtype=float)
        high = np.asarray(layout.get("high", (10.0, 10.0, 8.0)), dtype=float)
        rng = np.random.default_rng(seed)
        pos = rng.uniform(low, high, (count, 3))
        yaw = rng.uniform(-np.pi, np.pi, count)
    else:
        raise ValidationError(f"unknown layout kind {kind!r}")
    return pos, yaw
