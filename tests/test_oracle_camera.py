"""Pins for the oracle's ray generation (step a1, reading Q5: pinhole through pixel centres,
OpenGL axes x right / y up / -z forward, row 0 at the TOP, unit direction; include/plenoct.h
po_camera).  The paper has no camera model of its own ("invented plumbing"), so the
pins are rays worked out by hand for cameras whose geometry is obvious; a y-flip, a pixel-corner
instead of pixel-centre offset, swapped fx/fy or cx/cy, or a transposed c2w fails one of them.
"""
import numpy as np
import pytest

import gen

S3 = 1.0 / np.sqrt(3.0)


def _cam(c2w, fx, fy, cx, cy):
    c2w = np.asarray(c2w, np.float64)
    return gen.camera_record(c2w, fx, fy, cx, cy)


def _ray(om, cam, W, H, i, j):
    r = om.camera_rays(cam, W, H).reshape(H, W, 6)
    return r[j, i, :3], r[j, i, 3:]


def test_identity_camera_centre_and_corners(oracle_mod):
    """Camera at (1, 2, 3) with the identity rotation (looks down -z, y up), 5x5 pixels, f = 2,
    principal point at the image centre (2.5, 2.5): the centre pixel (2, 2) looks straight down
    -z; pixel (0, 0) is the TOP-left one, so its direction is left (-x), up (+y), forward (-z):
    (-1, 1, -1)/sqrt(3) -- offsets (0.5 - 2.5)/2 = -1 in x and -(0.5 - 2.5)/2 = +1 in y."""
    om = oracle_mod
    cam = _cam([[1, 0, 0, 1], [0, 1, 0, 2], [0, 0, 1, 3]], 2.0, 2.0, 2.5, 2.5)
    want = {(2, 2): (0.0, 0.0, -1.0),
            (0, 0): (-S3, S3, -S3),     # top-left
            (4, 0): (S3, S3, -S3),      # top-right
            (0, 4): (-S3, -S3, -S3),    # bottom-left
            (4, 4): (S3, -S3, -S3)}     # bottom-right
    for (i, j), d in want.items():
        o, got = _ray(om, cam, 5, 5, i, j)
        np.testing.assert_allclose(o, (1.0, 2.0, 3.0), rtol=0, atol=0)
        np.testing.assert_allclose(got, d, rtol=0, atol=1e-15)


def test_rotated_camera_looks_along_plus_x(oracle_mod):
    """A camera looking along world +x with world +z up: its right axis is world -y, its up axis
    world +z and its backward (+z_cam) axis world -x, i.e. c2w columns (0,-1,0), (0,0,1), (-1,0,0).
    The centre ray is (1, 0, 0); the top-left pixel looks forward (+x), left (+y) and up (+z):
    (1, 1, 1)/sqrt(3)."""
    om = oracle_mod
    cam = _cam([[0, 0, -1, -4], [-1, 0, 0, 0.5], [0, 1, 0, 0.25]], 2.0, 2.0, 2.5, 2.5)
    _, d = _ray(om, cam, 5, 5, 2, 2)
    np.testing.assert_allclose(d, (1.0, 0.0, 0.0), atol=1e-15)
    o, d = _ray(om, cam, 5, 5, 0, 0)
    np.testing.assert_allclose(o, (-4.0, 0.5, 0.25), atol=0)
    np.testing.assert_allclose(d, (S3, S3, S3), atol=1e-15)
    _, d = _ray(om, cam, 5, 5, 4, 4)   # bottom-right: forward, right (-y), down (-z)
    np.testing.assert_allclose(d, (S3, -S3, -S3), atol=1e-15)


def test_anisotropic_focal_and_offset_principal_point(oracle_mod):
    """fx = 1, fy = 2, principal point (1, 0.5) on a 4x2 image: pixel (3, 1) has camera-space
    direction ((3.5 - 1)/1, -(1.5 - 0.5)/2, -1) = (2.5, -0.5, -1), norm sqrt(7.5); pixel (1, 0)
    has ((1.5 - 1)/1, -(0.5 - 0.5)/2, -1) = (0.5, 0, -1), norm sqrt(1.25)."""
    om = oracle_mod
    cam = _cam(np.eye(3, 4), 1.0, 2.0, 1.0, 0.5)
    _, d = _ray(om, cam, 4, 2, 3, 1)
    np.testing.assert_allclose(d, np.array([2.5, -0.5, -1.0]) / np.sqrt(7.5), atol=1e-15)
    _, d = _ray(om, cam, 4, 2, 1, 0)
    np.testing.assert_allclose(d, np.array([0.5, 0.0, -1.0]) / np.sqrt(1.25), atol=1e-15)


@pytest.mark.parametrize("W,H", [(7, 3), (64, 64)])
def test_row_major_layout_and_unit_length(oracle_mod, W, H):
    """rays[(j * W + i)]: i runs along a row (x grows with i), rows go down the image (y falls
    with j); every direction is unit length; the origin is the camera position."""
    om = oracle_mod
    cam = _cam(np.eye(3, 4), 50.0, 50.0, W / 2.0, H / 2.0)
    r = om.camera_rays(cam, W, H).reshape(H, W, 6)
    np.testing.assert_allclose(np.linalg.norm(r[..., 3:], axis=-1), 1.0, atol=1e-15)
    assert np.all(np.diff(r[..., 3], axis=1) > 0)   # x increases along a row
    assert np.all(np.diff(r[..., 4], axis=0) < 0)   # y decreases down the columns
    assert np.all(r[..., :3] == 0.0)
