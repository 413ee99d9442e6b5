"""Host mapping rows (attachment_triplets, reference collision.py:430-462) on CPU."""

import numpy as np
import pytest

from paper_2306_06946_b200.collision import AttachKind, Attachment, attachment_triplets
from paper_2306_06946_b200.errors import InvalidAttachmentError


def test_vertex_and_barycentric_rows():
    r, c, v = attachment_triplets(Attachment(AttachKind.VERTEX, 0, vertex=4), 30, 6)
    assert (r, c, v) == ([6, 7, 8], [12, 13, 14], [1.0, 1.0, 1.0])
    att = Attachment(AttachKind.BARYCENTRIC, 0, triangle=np.array([2, 0, 7]), weights=np.array([0.2, 0.5, 0.3]))
    r, c, v = attachment_triplets(att, 30, 3)
    assert r == [3, 4, 5] * 3
    assert c == [6, 7, 8, 0, 1, 2, 21, 22, 23]
    assert v == [0.2] * 3 + [0.5] * 3 + [0.3] * 3


def test_rigid_lever_rows():
    lever = np.array([0.1, -0.2, 0.0])
    r, c, v = attachment_triplets(Attachment(AttachKind.RIGID_LOCAL, 0, lever=lever), 6, 0)
    J = np.zeros((3, 6))
    J[r, c] = v
    skew = np.array([[0.0, -lever[2], lever[1]], [lever[2], 0.0, -lever[0]], [-lever[1], lever[0], 0.0]])
    assert np.array_equal(J, np.hstack([np.eye(3), -skew]))
    assert len(v) == 3 + 4  # zero entries of the lever block are not stored


def test_out_of_range_and_dofless_kinds():
    with pytest.raises(InvalidAttachmentError):
        attachment_triplets(Attachment(AttachKind.VERTEX, 0, vertex=10), 30, 0)
    with pytest.raises(InvalidAttachmentError):
        attachment_triplets(Attachment(AttachKind.BARYCENTRIC, 0, triangle=np.array([0, 1, 10]),
                                       weights=np.ones(3) / 3), 30, 0)
    with pytest.raises(InvalidAttachmentError):
        attachment_triplets(Attachment(AttachKind.RIGID_LOCAL, 0, lever=np.zeros(3)), 30, 0)
    with pytest.raises(InvalidAttachmentError):
        attachment_triplets(Attachment(AttachKind.WORLD, 0, world_point=np.zeros(3)), 30, 0)


def test_rigid_mapping_rows():
    """S for a sphere-plane pair (collision.py:290-316, rows collision.py:448-457):
    [I, -skew(lever)], the plane side carrying no DoFs."""
    import paper_2306_06946_b200 as cn

    sph = cn.SphereGeometry(0, np.array([0.0, 0.05, 0.0]), 0.05, cn.Pose(np.eye(3), np.array([0.0, 0.05, 0.0])))
    pairs = cn.detect([sph, cn.PlaneGeometry(1, np.array((0.0, 1.0, 0.0)), 0.0)], 0.01)
    assert len(pairs) == 1 and pairs[0].attach_a.kind == cn.AttachKind.RIGID_LOCAL
    S = cn.build_signed_mapping(pairs, 0, 6).csr.toarray()
    lever = np.array([0.0, -0.05, 0.0])
    skew = np.array([[0.0, -lever[2], lever[1]], [lever[2], 0.0, -lever[0]], [-lever[1], lever[0], 0.0]])
    assert np.array_equal(S, np.hstack([np.eye(3), -skew]))
