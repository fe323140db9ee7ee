import sys, numpy as np, torch
sys.path.insert(0, ".")
import concurrent.futures as cf
import paper_2510_11508_b200 as nb
from paper_2510_11508_b200 import scenes
from torch.profiler import profile, ProfilerActivity
def gen(i):
    m = scenes.config5_map(i); return m.normals, m.mask, m.intrinsics()
if __name__ == "__main__":
    with cf.ProcessPoolExecutor(16) as ex: maps = list(ex.map(gen, range(64)))
    n = torch.from_numpy(np.stack([m[0] for m in maps])).cuda(); mk = torch.from_numpy(np.stack([m[1] for m in maps])).cuda()
    intr = [nb.CameraIntrinsics(*m[2]) for m in maps]
    nb.run_pipeline_batch(nb.NormalMap.create(n, mk), intr, float(np.deg2rad(3.5))); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        nb.run_pipeline_batch(nb.NormalMap.create(n, mk), intr, float(np.deg2rad(3.5))); torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=60))
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    span = ev[-1].time_range.end - ev[0].time_range.start
    fill = [e for e in ev if "fill_cg" in e.name]
    fe = fill[0].time_range.end
    post = [e for e in ev if e.time_range.start >= fe]
    pb = sum(e.time_range.end - e.time_range.start for e in post)
    ps = post[-1].time_range.end - fe
    print(f"span {span/1e3:.1f} ms busy {busy/1e3:.1f} ms; after fill: span {ps/1e3:.1f} ms busy {pb/1e3:.1f} ms, {len(post)} kernels/copies")
