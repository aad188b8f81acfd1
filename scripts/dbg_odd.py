import sys; sys.path.insert(0, '.')
from tests.test_gpu_parity import test_gpu_fp32_variant_scaled as t
t("c5", (17, 13, 6, 5, 11), 6); print("ok")
