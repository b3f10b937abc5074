import sys, numpy as np, torch
sys.path.insert(0, '.')
from scipy import ndimage
from oracle import stereonorm_oracle as orc
from paper_2504_15121_b200 import device, scenes
sc = scenes.street_scene(2048, 1024)
d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], 1.0, 3)
holes = ndimage.binary_dilation(np.random.default_rng(1003).random(d.shape) < 0.002, iterations=3)
d[holes] = np.nan
d = d.astype(np.float32)
rig = orc.Rig(sc.rig.fx, sc.rig.fy, sc.rig.u0, sc.rig.v0, sc.rig.baseline)
dt = torch.from_numpy(d).cuda()
for t in (0.05, 0.2, 1.0):
    P = orc.passable(d.astype(np.float64), rig, t)
    pg = device.passable(dt, sc.rig, t)[0].cpu().numpy().astype(bool)
    print("t", t, "passable equal", np.array_equal(P, pg), "count", P.sum())
    ref = orc.label_components(P)
    for trial in range(8):
        lab = device.component_labels(dt, sc.rig, t)[0].cpu().numpy().astype(np.int64)
        lab2 = device.labels_from_passable(torch.from_numpy(P).cuda())[0].cpu().numpy().astype(np.int64)
        bad = np.argwhere(lab != ref)
        bad2 = np.argwhere(lab2 != ref)
        print("  trial", trial, "mismatch", len(bad), "from_passable mismatch", len(bad2))
        if len(bad):
            y, x = bad[0]
            print("   first", (y, x), "got", lab[y, x], "want", ref[y, x], "P", P[y, x], "neg got", (lab[bad[:,0], bad[:,1]] < 0).sum())
            ys, xs = bad[:, 0], bad[:, 1]
            print("   y%64==0", np.mean(ys % 64 == 0), "x%32==0", np.mean(xs % 32 == 0), "distinct got", len(np.unique(lab[ys, xs])), "distinct want", len(np.unique(ref[ys, xs])))
