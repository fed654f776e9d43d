"""Write / read throughput of 64 MiB checkpoint-sized files on the box's
scratch disk: buffered (page cache, what the file stage uses), buffered with
fsync, and O_DIRECT.  Eight files in a row, like a pass's boundary stores."""
import json
import mmap
import os
import sys
import time

d = sys.argv[1] if len(sys.argv) > 1 else "/tmp/ackpt_disk_probe"
os.makedirs(d, exist_ok=True)
S = 64 << 20
buf = mmap.mmap(-1, S)  # page-aligned
buf.write(os.urandom(1 << 20) * 64)
out = {}
for mode in ("buffered", "buffered_fsync", "o_direct"):
    ts = []
    for i in range(8):
        path = os.path.join(d, f"f{i}.bin")
        flags = os.O_WRONLY | os.O_CREAT | os.O_TRUNC | (os.O_DIRECT if mode == "o_direct" else 0)
        t0 = time.perf_counter()
        fd = os.open(path, flags, 0o644)
        os.write(fd, buf)
        if mode == "buffered_fsync":
            os.fsync(fd)
        os.close(fd)
        ts.append(time.perf_counter() - t0)
    out[mode + "_write_gbs"] = [round(S / t / 1e9, 2) for t in ts]
t0 = time.perf_counter()
for i in range(8):
    with open(os.path.join(d, f"f{i}.bin"), "rb") as fh:
        fh.readinto(buf)
out["read_cached_gbs"] = round(8 * S / (time.perf_counter() - t0) / 1e9, 2)
for i in range(8):
    os.remove(os.path.join(d, f"f{i}.bin"))
st = os.statvfs(d)
out["fs_free_gb"] = round(st.f_bavail * st.f_frsize / 1e9, 1)
print(json.dumps(out))
