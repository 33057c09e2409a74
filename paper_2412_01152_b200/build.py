"""Build the in-tree CUDA library (sm_100a) and the CPU checkers."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def build_product() -> str:
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc")], check=True)
    return os.path.join(HERE, "libemesh_b200.so")


def build_oracle() -> None:
    # liboracle.so always; oracle/_ref only where the reference sources exist
    targets = ["all"] if os.path.isdir("/root/reference/proj/include/emesh") else [
        os.path.join(ROOT, "oracle", "liboracle.so")]
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), *targets], check=True)


def build_cpp_checks() -> None:
    # the C++ drop-in check compiles against the reference headers (this container only)
    if os.path.isdir("/root/reference/proj/include/emesh"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


if __name__ == "__main__":
    build_product()
    build_oracle()
    build_cpp_checks()
