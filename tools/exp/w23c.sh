cd /root/repo
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:pix" python tools/exp/w23.py 5 1 2>&1 | grep "pix_\|pixel_kernel" | head
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:pix" python tools/exp/w23.py 5 0 2>&1 | grep "pix_\|pixel_kernel" | head
python - <<'PY'
import numpy as np
a=np.load("/tmp/pix_5_0.npz"); b=np.load("/tmp/pix_5_1.npz")
np.set_printoptions(precision=17)
print(a["bd"][0,:2], b["bd"][0,:2])
PY
