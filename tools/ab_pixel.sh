cd /root/repo
python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectories.py tests/test_gpu_edges.py tests/test_gpu_large.py -q -x 2>&1 | tail -3
for cfg in "4 256" "2 1" "5 1"; do set -- $cfg
  for ty in 1 2; do for pw in 4 8; do
    echo "== cfg$1 S=$2 TY=$ty warps=$pw"
    PDF_PIX_TY=$ty PDF_PIX_WARPS=$pw python tools/timeline.py --cfg $1 --scenes $2 2>&1 | grep -E "period|^pixel "
  done; done
done
