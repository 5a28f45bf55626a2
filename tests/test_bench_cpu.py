"""bench.py host logic that runs without a GPU: the clock sampler's summary
(throttle reasons decoded from NVML bit rows and nvidia-smi rows alike)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench


def _sampler(rows, source):
    c = bench.ClockSampler(0)
    c.rows = rows
    c.source = source
    return c


def test_clock_summary_nvml_rows():
    na, ac = "Not Active", "Active"
    rows = [["1965", "1965", "", "0x0", na, na, na, na],
            ["1950", "1965", "", "0x4", na, na, na, ac],
            ["1965", "1965", "", "0x0", na, na, na, na]]
    s = _sampler(rows, "nvml").summary()
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]
    assert s["samples"] == 3 and s["source"] == "nvml"


def test_clock_summary_smi_rows_and_empty():
    rows = [["1800", "1965", "700.1", "0x0000000000000040", "Not Active", "Active", "Not Active", "Not Active"]]
    s = _sampler(rows, "nvidia-smi").summary()
    assert s["sm_mhz"] == 1800.0 and s["reasons"] == ["hw_thermal_slowdown"]
    assert _sampler([], None).summary()["reasons"] == ["unsampled"]


def test_clock_sampler_without_gpu_returns():
    # no NVML device / nvidia-smi here: the context must not hang and must
    # report the region as unsampled rather than invent clocks
    c = bench.ClockSampler(0)
    with c:
        pass
    s = c.summary()
    assert s["reasons"] == ["unsampled"] or s["samples"] >= 1


def test_gpus_flag_must_match_world_size():
    """bench.py --gpus N under a launcher whose WORLD_SIZE differs refuses to
    run (a scaling point must not silently measure another rank count)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "--gpus 4 but WORLD_SIZE=2" in r.stderr
