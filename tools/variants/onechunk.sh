python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "one_chunk_inf or ragged_chunk" 2>&1 | grep -E "assert|Error|passed|failed" | head -8
cp tools/variants/attn_tc_55838f5.cu paper_1910_01578_b200/csrc/attn_tc.cu
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
echo "--- old kernel"
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "one_chunk_inf or ragged_chunk" 2>&1 | grep -E "assert|Error|passed|failed" | head -8
