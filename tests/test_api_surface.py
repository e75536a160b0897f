"""The public names of the reference modules on the path (`hashsdf/*.py`, listed
here so the check runs without /root/reference) all exist in the package.  CPU only.
The reference's own small reverse-mode graph engine (`autodiff_oracle.py:22-205`) is
replaced by torch.autograd as the generic side of the Theorem-1 benchmark."""

from __future__ import annotations

import importlib

import pytest

REFERENCE_API = {
    "hash_encoding": ['CornerRecords', 'EncodedPoint', 'MultiResHashGrid', 'active_level_count', 'backward_first', 'backward_second', 'encode', 'encode_features_only', 'encode_jacobian', 'hash_index', 'hessian_contract', 'level_resolutions'],
    "relu_mlp": ['ForwardTrace', 'MlpWeights', 'ShapeError', 'backward_first', 'backward_second', 'backward_second_row', 'forward', 'input_jacobian', 'input_jacobian_rows', 'second_order_input_residual'],
    "field": ['FieldCache', 'FieldConfig', 'FieldGrads', 'SdfFieldParams', 'eval_color', 'eval_field', 'eval_normal', 'eval_sdf', 'field_backward', 'sal_geometry_init', 'sigmoid'],
    "renderer": ['MarchResult', 'OccupancyGrid', 'RenderRecords', 'alpha', 'backward_cotangents', 'composite', 'expected_depth', 'field_sdf_only', 'intersect_aabb', 'march_rays', 'render_rays', 'sdf_transforms', 'update_occupancy'],
    "trainer": ['AdamState', 'LossReport', 'TrainConfig', 'TrainResult', 'TrainState', 'adam_update', 'apply_gradients', 'color_loss', 'compute_cotangents', 'eikonal_loss', 'evaluate_view', 'huber', 'huber_grad', 'level_schedule', 'lr_factor', 'masked_psnr', 'psnr', 'render_frame', 'train_static', 'train_step'],
    "scene_io": ['CameraFrame', 'MultiViewDataset', 'RayBatch', 'generate_ray', 'generate_rays_grid', 'load_dataset', 'make_synthetic', 'preset_scene', 'project_point', 'sample_ray_batch', 'scene_sdf'],
    "checkpoint": ['load_checkpoint', 'read_sections', 'save_checkpoint'],
    "_kernels": ['adam_step', 'hessian_contract', 'interp_features', 'interp_full', 'scatter_first', 'scatter_second'],
    "autodiff_oracle": ['bench_rows_to_csv', 'bench_second_order'],
}


@pytest.mark.parametrize("module", sorted(REFERENCE_API))
def test_reference_names_exist(module):
    mod = importlib.import_module(f"paper_2212_05231_b200.{module}")
    missing = [n for n in REFERENCE_API[module] if not hasattr(mod, n)]
    assert not missing, f"{module}: {missing}"
