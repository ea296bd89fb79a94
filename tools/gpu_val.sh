cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -q -m gpu --timeout 2300 -p no:cacheprovider 2>&1 | tail -4
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
