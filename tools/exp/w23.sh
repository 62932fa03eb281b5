cd /root/repo
for c in 4 5; do for s in 0 1; do python tools/exp/w23.py $c $s; done; done
python - <<'PY'
import numpy as np
for c in (4,5):
    a=np.load(f"/tmp/pix_{c}_0.npz"); b=np.load(f"/tmp/pix_{c}_1.npz")
    ga=np.abs(a["ga"]-b["ga"]).reshape(a["ga"].shape[0],-1).max(1)/np.abs(a["ga"]).reshape(a["ga"].shape[0],-1).max(1)
    print("cfg",c,"g_alpha max rel diff per scene: max",ga.max(),"median",np.median(ga))
    print("   breakdown rel diff (state,data,bound,tv,bridge,total):",np.abs(a["bd"]-b["bd"]).max(0)/np.abs(a["bd"]).max(0))
    print("   state/total:", (a["bd"][:,0]/a["bd"][:,5]).min(), (a["bd"][:,0]/a["bd"][:,5]).max())
PY
