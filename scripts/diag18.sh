O=gpurun_out/diag18; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "group or stream or linear" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 300 python scripts/kbench.py --cases gate_8b,down_8b,gateup_8b,gateup_1b,down_1b,qkv_1b,lmhead_8b --routes 0,1 > $O/kb.txt 2>&1
