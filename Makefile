# Builds the C-ABI library for B200 (sm_100a): objects compiled in parallel, then linked.
# Same as `python -c "import __graft_entry__ as g; g.build()"`.
PY ?= python
.PHONY: lib bounds clean
lib:
	$(PY) -c "import __graft_entry__ as g; g.build()"
bounds:
	$(PY) -c "import __graft_entry__ as g; g.build(variant='bounds')"
clean:
	rm -rf paper_2003_07065_b200/_build paper_2003_07065_b200/libsst*.so build_ptxas*.log
