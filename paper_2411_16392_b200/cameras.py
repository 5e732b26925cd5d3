"""Pinhole camera type used at the rasterizer boundary.

Mirrors qgsplat.cameras.Camera (/root/reference/pkg/src/qgsplat/cameras.py:15-94):
OpenCV frame (x right, y down, z forward); the ray of pixel (u, v) passes
through ((u+0.5-cx)/fx, (v+0.5-cy)/fy, 1); depth is Euclidean distance along
the unit ray.  Any object with the same attributes (fx, fy, cx, cy, width,
height, world_to_camera) is accepted by the rasterizer, including the
reference's own Camera.
"""

from dataclasses import dataclass

import numpy as np


@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    world_to_camera: np.ndarray
    image: str = ""

    def __post_init__(self):
        self.world_to_camera = np.asarray(self.world_to_camera, dtype=np.float64)
        if self.world_to_camera.shape != (4, 4):
            raise ValueError("world_to_camera must be 4x4")
        if not (self.fx > 0 and self.fy > 0):
            raise ValueError("focal lengths must be positive")
        R = self.R_wc
        if np.abs(R @ R.T - np.eye(3)).max() > 1e-6:
            raise ValueError("world_to_camera rotation is not orthonormal")

    @property
    def R_wc(self):
        return self.world_to_camera[:3, :3]

    @property
    def t_wc(self):
        return self.world_to_camera[:3, 3]

    @property
    def R_cw(self):
        return self.R_wc.T

    @property
    def center(self):
        return -self.R_wc.T @ self.t_wc

    def to_cam(self, pts_world):
        return np.asarray(pts_world, dtype=np.float64) @ self.R_wc.T + self.t_wc

    def project(self, pts_world):
        pc = self.to_cam(pts_world)
        z = pc[..., 2]
        return self.fx * pc[..., 0] / z + self.cx, self.fy * pc[..., 1] / z + self.cy, z

    def ray_world(self, u, v):
        d = np.array([(u + 0.5 - self.cx) / self.fx, (v + 0.5 - self.cy) / self.fy, 1.0])
        d /= np.linalg.norm(d)
        return self.center, self.R_cw @ d


def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """world_to_camera for a camera at eye looking at target (cameras.py:97-111)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    if np.linalg.norm(right) < 1e-8:
        right = np.cross(fwd, np.array([0.0, 1.0, 0.0]))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    w2c = np.eye(4)
    w2c[:3, :3] = np.stack([right, down, fwd])
    w2c[:3, 3] = -w2c[:3, :3] @ eye
    return w2c
