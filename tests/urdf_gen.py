"""Random URDF documents for parity tests (the URDF analogue of
proj/tests/helpers.hpp:124-150 random_tree), including fixed joints, prismatic
joints, general axes and inertial rpy so every loader/packer path is hit."""
import numpy as np


def _vec(v):
    return " ".join(repr(float(x)) for x in v)


def random_urdf(seed, n=10, branchiness=0.5, fixed_prob=0.2, axis_aligned_prob=0.4):
    rng = np.random.default_rng(seed)
    links, joints = [], []

    def inertial(name):
        m = rng.uniform(0.2, 3.0)
        a = rng.uniform(-1, 1, (3, 3))
        I = 0.05 * (a @ a.T + 0.02 * np.eye(3))
        com = rng.uniform(-0.15, 0.15, 3)
        rpy = rng.uniform(-np.pi, np.pi, 3) if rng.uniform() < 0.3 else np.zeros(3)
        return (f'  <link name="{name}">\n    <inertial>\n      <origin xyz="{_vec(com)}" rpy="{_vec(rpy)}"/>\n'
                f'      <mass value="{float(m)!r}"/>\n'
                f'      <inertia ixx="{float(I[0,0])!r}" ixy="{float(I[0,1])!r}" ixz="{float(I[0,2])!r}" iyy="{float(I[1,1])!r}" '
                f'iyz="{float(I[1,2])!r}" izz="{float(I[2,2])!r}"/>\n    </inertial>\n  </link>\n')

    links.append(inertial("link0"))
    for i in range(1, n + 1):
        links.append(inertial(f"link{i}"))
        parent = i - 1
        if i > 1 and rng.uniform() < branchiness:
            parent = int(rng.integers(0, i - 1))
        u = rng.uniform()
        jtype = "fixed" if u < fixed_prob else ("prismatic" if u < fixed_prob + 0.15 else
                                                 ("continuous" if rng.uniform() < 0.2 else "revolute"))
        if rng.uniform() < axis_aligned_prob:
            axis = np.zeros(3)
            axis[int(rng.integers(0, 3))] = 1.0 if rng.uniform() < 0.7 else -1.0
        else:
            axis = rng.normal(size=3)
            axis /= np.linalg.norm(axis)
        xyz = rng.uniform(-0.4, 0.4, 3)
        rpy = rng.uniform(-np.pi, np.pi, 3)
        extra = f'\n    <axis xyz="{_vec(axis)}"/>' if jtype != "fixed" else ""
        joints.append(f'  <joint name="j{i:03d}" type="{jtype}">\n    <parent link="link{parent}"/>\n'
                      f'    <child link="link{i}"/>\n    <origin xyz="{_vec(xyz)}" rpy="{_vec(rpy)}"/>{extra}\n'
                      f'  </joint>\n')
    # a massless tool frame on the last link
    links.append('  <link name="tool"/>\n')
    joints.append(f'  <joint name="zz_tool" type="fixed">\n    <parent link="link{n}"/>\n    <child link="tool"/>\n'
                  f'    <origin xyz="0.1 0.02 -0.03" rpy="0.3 -0.2 0.1"/>\n  </joint>\n')
    return '<?xml version="1.0"?>\n<robot name="random">\n' + "".join(links) + "".join(joints) + "</robot>\n"
