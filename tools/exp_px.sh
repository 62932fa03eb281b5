cd /root/repo
echo "cfg5"; python tools/phases.py --cfg 5 --iters 5 2>&1 | tail -1 | cut -c60-330
python -m pytest tests/test_gpu_large.py -x -q 2>&1 | tail -1
sed -i 's/__launch_bounds__(256, (E >= 4 ? 2 : 1)) vl_cols_kernel/__launch_bounds__(256) vl_cols_kernel/' paper_2602_13805_b200/csrc/pdf_view_large.cuh
python -m paper_2602_13805_b200.build > /dev/null 2>&1
echo "cfg5 no-minblocks"; python tools/phases.py --cfg 5 --iters 5 2>&1 | tail -1 | cut -c60-330
