"""Which NVML NVLink traffic counters move on this box? Copies 8 GiB cuda:0 -> cuda:1
over peer access and prints, per candidate field id, the per-GPU delta summed over
active links (and nvidia-smi nvlink -gt d before/after). Needs 2 GPUs."""
import subprocess
import sys

import pynvml as N
import torch

FIELDS = {138: "THROUGHPUT_DATA_TX(KiB)", 139: "THROUGHPUT_DATA_RX(KiB)", 140: "THROUGHPUT_RAW_TX(KiB)",
          141: "THROUGHPUT_RAW_RX(KiB)", 201: "COUNT_XMIT_PACKETS", 202: "COUNT_XMIT_BYTES",
          203: "COUNT_RCV_PACKETS", 204: "COUNT_RCV_BYTES"}


def read(h, links, scope_all):
    out = {}
    for f in FIELDS:
        tot, errs = 0, set()
        scopes = [0xFFFFFFFF] if scope_all else links
        for l in scopes:
            v = N.nvmlDeviceGetFieldValues(h, [(f, l)])[0]
            if v.nvmlReturn != 0:
                errs.add(v.nvmlReturn)
                continue
            tot += v.value.ullVal
        out[f] = (tot, sorted(errs))
    return out


def main():
    N.nvmlInit()
    hs = [N.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
    links = []
    for h in hs:
        ls = []
        for l in range(18):
            try:
                if N.nvmlDeviceGetNvLinkState(h, l) == 1:
                    ls.append(l)
            except N.NVMLError:
                pass
        links.append(ls)
    print("active links", [len(l) for l in links])
    smi0 = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True).stdout
    a = torch.empty(1 << 31, dtype=torch.float32, device="cuda:0").fill_(1.0)
    b = torch.empty_like(a, device="cuda:1")
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    before = {(g, s): read(hs[g], links[g], s) for g in range(2) for s in (False, True)}
    for _ in range(1):
        b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    after = {(g, s): read(hs[g], links[g], s) for g in range(2) for s in (False, True)}
    smi1 = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True).stdout
    print(f"copied {a.numel() * 4} bytes cuda:0 -> cuda:1")
    for (g, s), v in after.items():
        for f, (tot, errs) in v.items():
            d = tot - before[(g, s)][f][0]
            print(f"gpu{g} {'scope=all' if s else 'per-link'} field {f} {FIELDS[f]}: delta {d} errs {errs}")
    print("nvidia-smi before:\n" + smi0[:3000])
    print("nvidia-smi after:\n" + smi1[:3000])
    return 0


if __name__ == "__main__":
    sys.exit(main())
