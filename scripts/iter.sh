#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/e2e_phases.py 2>&1 | tail -12
