"""Read-only NVML probe of the SYnergy clock controls on a GPU box.

    python scripts/nvml_probe.py [device]

Prints the supported SM clocks, the current / default application clocks,
the API-restriction state of the clock setters and the energy counter.  It
never changes a clock (the pool's operators forbid clock changes; the
driver resets and records them), so it is the evidence behind DESIGN.md §7.
"""
import json
import sys

import pynvml as nv


def main():
    dev = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(dev)
    out = {"name": nv.nvmlDeviceGetName(h), "driver": nv.nvmlSystemGetDriverVersion()}

    def q(key, fn, *a):
        try:
            v = fn(*a)
            out[key] = v
        except nv.NVMLError as exc:  # noqa: PERF203
            out[key] = f"NVMLError: {exc}"

    q("supported_mem_mhz", nv.nvmlDeviceGetSupportedMemoryClocks, h)
    mem = out["supported_mem_mhz"][0] if isinstance(out["supported_mem_mhz"], list) else None
    if mem is not None:
        q("supported_sm_mhz", nv.nvmlDeviceGetSupportedGraphicsClocks, h, mem)
    q("app_sm_mhz", nv.nvmlDeviceGetApplicationsClock, h, nv.NVML_CLOCK_SM)
    q("default_app_sm_mhz", nv.nvmlDeviceGetDefaultApplicationsClock, h, nv.NVML_CLOCK_SM)
    q("max_sm_mhz", nv.nvmlDeviceGetMaxClockInfo, h, nv.NVML_CLOCK_SM)
    q("cur_sm_mhz", nv.nvmlDeviceGetClockInfo, h, nv.NVML_CLOCK_SM)
    q("power_limit_mw", nv.nvmlDeviceGetPowerManagementLimit, h)
    q("energy_mj", nv.nvmlDeviceGetTotalEnergyConsumption, h)
    q("api_restriction_app_clocks", nv.nvmlDeviceGetAPIRestriction, h,
      nv.NVML_RESTRICTED_API_SET_APPLICATION_CLOCKS)
    q("api_restriction_auto_boost", nv.nvmlDeviceGetAPIRestriction, h,
      nv.NVML_RESTRICTED_API_SET_AUTO_BOOSTED_CLOCKS)
    q("persistence_mode", nv.nvmlDeviceGetPersistenceMode, h)
    sm = out.get("supported_sm_mhz")
    if isinstance(sm, list):
        out["n_supported_sm_clocks"] = len(sm)
        out["supported_sm_mhz"] = sorted(sm, reverse=True)
    print(json.dumps(out, indent=1, default=str))
    nv.nvmlShutdown()


if __name__ == "__main__":
    main()
