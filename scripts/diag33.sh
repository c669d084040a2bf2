O=gpurun_out/diag33; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 200 python scripts/kbench.py --cases up_3b_m16,up_3b_m64,q_3b_m64,lmhead_8b_m16,lmhead_8b_m64 --routes 0,1 > $O/kb.txt 2>&1
