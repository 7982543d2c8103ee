"""Small helpers shared by the tests (test infrastructure)."""


def camera_from_record(rec):
    from paper_2406_11836_b200.capi import Camera
    return Camera.from_record(rec)
