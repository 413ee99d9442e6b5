"""Host-side scene logic without a GPU: the Newton iteration count a step
without contacts reports, as the reference's loop (solver.py:260-367) counts
it on empty pairs (StepReport.newton_iterations = len(result.iterations),
scene.py:744)."""

from paper_2306_06946_b200.scene import _contactless_iterations
from paper_2306_06946_b200.solver import NewtonConfig


def test_contactless_iteration_counts():
    # defaults: pen 0 <= 1e-5 stops after the first iteration
    assert len(_contactless_iterations(NewtonConfig(scheme="fast", max_iterations=5))) == 1
    # forced iterations: every iteration runs an empty PGS
    forced = NewtonConfig(scheme="fast", max_iterations=5, penetration_tol=-1.0, rotation_tol=-1.0)
    its = _contactless_iterations(forced)
    assert len(its) == 5 and all(i.pgs_iterations == 0 and i.penetration == 0.0 for i in its)
    # forced penetration, default rotation tolerance: the zero rotation stops iteration 2
    assert len(_contactless_iterations(NewtonConfig(scheme="fast", max_iterations=5, penetration_tol=-1.0))) == 1
    # no re-linearisation: only the penetration test stops the loop
    nr = NewtonConfig(scheme="standard", max_iterations=4, penetration_tol=-1.0, relinearize=False)
    assert len(_contactless_iterations(nr)) == 4
    assert len(_contactless_iterations(NewtonConfig(scheme="single", max_iterations=7, penetration_tol=-1.0))) == 1
