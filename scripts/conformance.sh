#!/bin/bash
# The reference's OWN unit/acceptance tests run unchanged against the drop-in through an
# `otmatch` alias (tests/conformance/otmatch -> paper_2111_05366_b200 -> libgoat.so).
# The test files are staged, unmodified, by __graft_entry__.build() into the git-ignored
# baseline/_ref/tests/ (only where /root/reference exists); they are never committed.
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
if [ ! -d baseline/_ref/tests ]; then echo "baseline/_ref/tests missing: run python -c 'import __graft_entry__ as g; g.stage_reference_tests()' where /root/reference exists"; exit 2; fi
PYTHONPATH=tests/conformance:. timeout ${CONF_TIMEOUT:-1500} python -m pytest baseline/_ref/tests -q -p no:cacheprovider -rs "$@"
