"""The drop-in switch: route the reference package's hot-path entry points to this build.

A `splatslam` maintainer opts in from `splatslam/__init__.py`:

    if os.environ.get("SPLATSLAM_BACKEND") == "b200":
        import paper_2507_04004_b200.dropin
        paper_2507_04004_b200.dropin.install(sys.modules[__name__])

`install(pkg)` rebinds, in the package's own submodules, exactly the names below -- the reference
callers (`optimize_map` R/mapper.py:246-257, `expand_map` :218-230, `photometric_refine`
R/odometry.py:305-336, `_render_map_view` R/cli.py:155, `interpolate_frames` R/apps.py:221) look
them up through those modules, so they reach the sm_100a kernels with no other change.  Argument
meaning, return types and error taxonomy follow the reference: with the reference's own numpy
`GaussianMap`, results come back as numpy arrays and `sparse_adam_step` / `optimize_map` update
the caller's arrays in place.  `install` returns the previous bindings; `uninstall(pkg, saved)`
restores them.
"""

from __future__ import annotations

import importlib

# (submodule, name) -> (our module, our name)
BINDINGS = {
    "rasterizer": {name: ("rasterizer", name) for name in (
        "forward", "backward", "backward_2d", "pose_backward", "cull_tiles", "sparse_adam_step", "AdamState",
        "default_lrs", "Camera", "RenderOutput")},                              # R/rasterizer.py:47-725
    "losses": {name: ("losses", name) for name in (
        "mapping_loss", "photometric_loss", "dssim_and_grad", "depth_ratio_loss")},  # R/losses.py:89-161
    "gaussians": {"project": ("gaussians", "project"), "eval_sh": ("gaussians", "eval_sh"),  # :102-215
                  "init_from_points": ("gaussians", "init_from_points"),       # R/gaussians.py:227-248
                  "save_gaussian_ply": ("mapio", "save_gaussian_ply"),         # R/gaussians.py:257-272
                  "load_gaussian_ply": ("mapio", "load_gaussian_ply")},        # R/gaussians.py:275-305
    "mapper": {**{name: ("mapper", name) for name in (
        "optimize_map", "project_points", "bilinear_color", "zbuffer_project", "group_mapping_data", "init_map",
        "expand_map", "Mapper", "mapping_loop")},                               # R/mapper.py:69-334
               "save_keyframe": ("archive", "save_keyframe"),                   # R/mapper.py:341-349
               "load_keyframe": ("archive", "load_keyframe")},                  # R/mapper.py:352-364
    "odometry": {"photometric_refine": ("odometry", "photometric_refine")},     # R/odometry.py:305-336
}


def install(pkg) -> dict:
    """Rebind the hot-path names of `pkg` (the splatslam package module) to this build; returns
    {(submodule, name): previous object} for `uninstall`."""
    from . import _lib
    saved = {("_lib", "HOST_ARRAYS"): _lib.HOST_ARRAYS}
    _lib.HOST_ARRAYS = True  # reference callers get numpy arrays from every entry point
    for sub, names in BINDINGS.items():
        target = importlib.import_module(f"{pkg.__name__}.{sub}")
        for name, (ours, ours_name) in names.items():
            impl = getattr(importlib.import_module(f"{__package__}.{ours}"), ours_name)
            saved[(sub, name)] = getattr(target, name, None)
            setattr(target, name, impl)
    return saved


def uninstall(pkg, saved: dict) -> None:
    from . import _lib
    _lib.HOST_ARRAYS = saved.pop(("_lib", "HOST_ARRAYS"), False)
    for (sub, name), obj in saved.items():
        target = importlib.import_module(f"{pkg.__name__}.{sub}")
        if obj is None:
            if hasattr(target, name):
                delattr(target, name)
        else:
            setattr(target, name, obj)
