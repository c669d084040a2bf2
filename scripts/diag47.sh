# final HEAD: full GPU suite + smoke (default dispatch)
O=gpurun_out/diag47; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
