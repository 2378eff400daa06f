"""The Python example of README.md runs as written (on a GPU)."""
import os
import re

import pytest

pytestmark = pytest.mark.gpu


def test_readme_python_example():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "README.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    assert blocks, "README has no python example"
    for code in blocks:
        exec(compile(code, "README.md", "exec"), {})
