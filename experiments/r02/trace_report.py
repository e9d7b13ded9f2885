"""Summarise LAM_STEP_TRACE stamps (bench.py, peer engine, step launch): per (layer, micro-batch)
launch: time waiting for inputs, attention, publication, and the relay back to the next layer."""
import glob
import sys

import numpy as np

d = sys.argv[1]
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for f in sorted(glob.glob(f"{d}/rank*.npy")):
    t = np.load(f).astype(np.float64).reshape(-1, mb, 4)  # [layer, mb, stamp]
    L = t.shape[0]
    t0 = t[:, :, 0].min()
    t = (t - t0) / 1000.0  # us
    seen, done, pub = t[:, :, 1], t[:, :, 2], t[:, :, 3]
    attn = done - seen                       # inputs seen -> last unit done
    pubd = pub - done                        # last unit -> flags published
    relay = seen[1:] - pub[:-1]              # layer l published -> layer l+1 inputs seen
    step = pub.max() - seen.min()
    print(f"{f}: step {step:.1f} us ({step / L:.1f} us/layer); per launch median: "
          f"attention {np.median(attn):.1f}, publish {np.median(pubd):.2f}, relay {np.median(relay):.1f} "
          f"(p90 {np.percentile(relay, 90):.1f}) us")
    for l in (0, 1, 2, L // 2, L - 1):
        print("   layer", l, " ".join(f"mb{m}: seen {seen[l, m]:.1f} done {done[l, m]:.1f} pub {pub[l, m]:.1f}"
                                      for m in range(mb)))

# per-CTA claim records (3 words each, 400 per CTA, first 1024 CTAs)
for f in sorted(glob.glob(f"{d}/rank*.npy"))[:1]:
    raw = np.load(f)
    n_lm = None
    for cand in (mb * 80, mb * 32, mb):
        pass
    base = raw[: len(raw) - 3 * 400 * 1024]
    n_lm = len(base) // 4
    recs = raw[len(base):].reshape(1024, 400, 3)
    valid = recs[:, :, 0] != -1
    ctas = int(valid.any(axis=1).sum())
    idx = recs[:, :, 2][valid]
    items_per_lm = (idx.max() + 1) // n_lm
    t0 = recs[:, :, 0][valid].min()
    waits, durs, first_wait = [], [], []
    for c in range(ctas):
        r = recs[c][valid[c]].astype(np.float64)
        if len(r) < 2:
            continue
        r[:, :2] = (r[:, :2] - t0) / 1000.0
        waits.append((r[:, 1] - r[:, 0]).sum())
        durs.extend(np.diff(r[:, 0]))
    span = (recs[:, :, 1][valid].max() - t0) / 1000.0
    w = np.array(waits)
    print(f"{f}: {ctas} CTAs, {items_per_lm} items per launch, recorded span {span:.0f} us; "
          f"input waits per CTA: mean {w.mean():.0f} us ({100 * w.mean() / span:.1f}% of span); "
          f"claim-to-claim median {np.median(durs):.1f} us, p10 {np.percentile(durs, 10):.1f}, p90 {np.percentile(durs, 90):.1f}")
    # the waits by launch lm (sum over CTAs, us) for a few layers in the middle
    lm_of = lambda i: min(int(i) // items_per_lm, n_lm - 1)  # noqa: E731  (approximate with splits)
    per_lm = np.zeros(n_lm)
    for c in range(ctas):
        r = recs[c][valid[c]]
        for a, b, i in r:
            per_lm[lm_of(i)] += (b - a) / 1000.0
    mid = n_lm // 2
    print("   summed CTA wait (us) by launch lm, middle:", " ".join(f"{x:.0f}" for x in per_lm[mid:mid + 8]))
