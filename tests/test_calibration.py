"""The measured-bandwidth predictor (paper_2412_16434_b200/calibrate.py):
profiles built from the committed B200 calibration drive the store's cost
model (transfer_time / decode_step_time, reference costmodel.cpp:59-95)."""
import json

from conftest import ROOT

from paper_2412_16434_b200 import calibrate
from paper_2412_16434_b200 import kvstore as K


def test_calibrated_profiles_drive_the_cost_model(product_libs):
    cal = json.loads((ROOT / "profiles" / "calibration_r01.json").read_text())
    links = calibrate.link_profile(cal)
    gpu = calibrate.gpu_profile(cal)
    # one 8B layer (512 x 64 KiB pages) over calibrated PCIe: tens of GB/s, not the reference's 25
    layer = 512 * 65536
    t = K.transfer_time(layer, K.PCIE_H2D, links)
    assert abs((t - links.per_transfer_latency) - layer / links.pcie_bandwidth * 1e9) <= 1
    assert links.pcie_bandwidth > 40e9
    # the decode step follows the measured curve, clamped at its ends
    curve = dict(cal["decode_curve_ms"])
    assert K.decode_step_time(1, gpu) == round(curve[1] * 1e6)
    assert K.decode_step_time(64, gpu) == round(curve[64] * 1e6)
    assert K.decode_step_time(512, gpu) == round(curve[64] * 1e6)
    st = K.KvStore(gpu=gpu, links=links)
    assert st.layer_block_bytes() == 65536
