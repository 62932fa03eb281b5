cd /root/repo
python - <<'PY'
import numpy as np
for c in (5,):
    a=np.load(f"/tmp/pix_{c}_0.npz"); b=np.load(f"/tmp/pix_{c}_1.npz")
    print(repr(a["bd"]), repr(b["bd"]))
PY
PDF_PIX_STREAM=0 python tools/timeline.py --cfg 5 2>&1 | grep "^pixel "
python tools/exp/w23.py 5 0; python tools/exp/w23.py 5 1
python - <<'PY'
import numpy as np
a=np.load("/tmp/pix_5_0.npz"); b=np.load("/tmp/pix_5_1.npz")
print(repr(a["bd"]), repr(b["bd"]))
PY
