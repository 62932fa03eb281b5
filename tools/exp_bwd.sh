cd /root/repo
for v in "4 4" "3 4" "3 8" "2 8"; do
  set -- $v
  sed -i "s/^constexpr int BM_D = [0-9];/constexpr int BM_D = $1;/; s/^constexpr int BM_WARPS = [0-9];/constexpr int BM_WARPS = $2;/" paper_2602_13805_b200/csrc/pdf_net_mma.cuh
  python -m paper_2602_13805_b200.build > /dev/null 2>&1 || echo BUILD FAIL
  echo "D=$1 W=$2"; python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c230-420
  python tools/phases.py --cfg 2 2>&1 | tail -1 | cut -c60-100
done
