"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no ray traversal, no SH
evaluation, no compositing).  It only produces the *inputs* of the hot path:

* PlenOctree arrays in the C-ABI layout of ``include/plenoct.h``
  (child table ``uint32[n_nodes][8]``, leaf ``sigma[n_leaves]`` (pre-ReLU
  sigma-tilde) and ``sh[n_leaves][B][3]``);
* cameras (``po_camera`` records) and ray batches;
* training targets for the optimisation step are produced by the *caller*
  (they are renders), never here.

Every random draw comes from numpy's counter-based Philox generator keyed by
an explicit seed, so the same call gives the same arrays on every machine.
The scene recipes are stated in DESIGN.md ("Input recipe").
"""
from .trees import (Tree, TAG_EMPTY, TAG_INTERNAL, TAG_LEAF, build_from_leaf_cells,
                    uniform_tree, random_tree, tree_leaf_boxes)
from .scenes import scene_c0, scene_c1, scene_c3, scene_random, make_payload_random
from .cameras import (camera_record, orbit_camera, config_camera, fibonacci_hemisphere,
                      random_rays, camera_rays_f32)

__all__ = [
    "Tree", "TAG_EMPTY", "TAG_INTERNAL", "TAG_LEAF", "build_from_leaf_cells", "uniform_tree",
    "random_tree", "tree_leaf_boxes", "scene_c0", "scene_c1", "scene_c3", "scene_random",
    "make_payload_random", "camera_record", "orbit_camera", "config_camera",
    "fibonacci_hemisphere", "random_rays", "camera_rays_f32",
]
